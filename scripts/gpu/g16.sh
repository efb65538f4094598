mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
timeout 900 python -m pytest tests/test_gpu_trsv_variants.py -x -q > gpurun_out/g16_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/g16_pytest.log
timeout 1500 python scripts/trsv_sweep.py --ls-p 4 --syncfree --env RSB_TRSV_GRID=static --env "RSB_TRSV_GRID=static;RSB_WIDE_N=4" > gpurun_out/g16_sweep.log 2>&1; echo sweep rc=$?
tail -c 2500 gpurun_out/g16_sweep.log
