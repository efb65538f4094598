mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
timeout 1500 python scripts/trsv_sweep.py --ls-p 4 --syncfree --env RSB_TRSV_EVICT=1 --env RSB_TRSV_PERSIST=1 --env "RSB_TRSV_EVICT=1;RSB_TRSV_PERSIST=1" > gpurun_out/g14_sweep.log 2>&1; echo sweep rc=$?
tail -c 3000 gpurun_out/g14_sweep.log
