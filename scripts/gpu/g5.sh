mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
timeout 600 python -m pytest tests/test_gpu_trsv_variants.py tests/test_gpu_batch.py -x -q > gpurun_out/g5_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/g5_pytest.log
timeout 1500 python bench.py --no-tol --no-parity > gpurun_out/g5_b8m.log 2>&1; echo b8m rc=$?
tail -c 2500 gpurun_out/g5_b8m.log
