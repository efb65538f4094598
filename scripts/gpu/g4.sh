mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q > gpurun_out/g4_pytest.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/g4_pytest.log
