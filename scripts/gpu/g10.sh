mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
timeout 900 python scripts/setup_timing.py 8000000 > gpurun_out/g10_setup.log 2>&1; echo rc=$?
cat gpurun_out/g10_setup.log | tail -30
