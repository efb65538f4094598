mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_illc1850.py tests/test_gpu_baseline_sizes.py -x -q --durations=15 -k "not config3" > gpurun_out/g9_pytest.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/g9_pytest.log
