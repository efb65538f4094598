mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
NCU=/usr/local/cuda/bin/ncu
timeout 900 python scripts/trsv_once.py > gpurun_out/g13_warm.log 2>&1; echo warm rc=$?
timeout 1500 $NCU --set full --clock-control none --import-source on -k regex:"k_trsv|k_wide|k_fill" -o gpurun_out/g13_trsv python scripts/trsv_once.py > gpurun_out/g13_ncu.log 2>&1; echo ncu rc=$?
$NCU -i gpurun_out/g13_trsv.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,lts__t_sector_hit_rate.pct,launch__registers_per_thread,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/g13_trsv_raw.csv 2>&1; echo raw rc=$?
timeout 1500 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/g13_launches.csv python bench.py --steps 2 --warmup 1 --no-tol --no-parity --batch 0 > gpurun_out/g13_bench_ncu.log 2>&1; echo launches rc=$?
ls -la gpurun_out/ | tail
