mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
timeout 600 python -m pytest tests/test_gpu_trsv_variants.py tests/test_gpu_configs.py -x -q > gpurun_out/g3_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/g3_pytest.log
timeout 1200 python scripts/trsv_sweep.py --ls-p 1,2,4 --occ 1 --syncfree > gpurun_out/g3_sweep.log 2>&1; echo sweep rc=$?
tail -c 3000 gpurun_out/g3_sweep.log
