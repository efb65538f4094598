mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
ls /tmp/rsb_fc 2>/dev/null | head
timeout 1200 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g6_launches.csv python scripts/batch_profile.py --n 8000000 --iters 2 > gpurun_out/g6.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/g6.log
wc -l gpurun_out/g6_launches.csv
