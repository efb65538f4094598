mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
timeout 900 python -m pytest tests/test_gpu_device_setup.py -x -q --durations=5 > gpurun_out/g11_pytest.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/g11_pytest.log
timeout 900 python scripts/setup_timing.py 8000000 > gpurun_out/g11_setup.log 2>&1; echo rc=$?
tail -8 gpurun_out/g11_setup.log
