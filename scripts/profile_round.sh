#!/bin/bash
# Measurement pass for profiles/ (run on the GPU box through gpurun, from the
# repo root).  Each ncu command runs only after the same command exited 0
# without ncu.  Outputs go to gpurun_out/prof/; scripts/summarize_profiles.py
# turns them into the profiles/ files.
#
#   config 1 (the BASELINE workload, bench.py's default): bench line, the
#     reference arm, the ncu launch list of a short run, ncu --set full of the
#     8 triangular solves of one timed iteration
#   config 4 structure: the full-size (n = 8e6) bench line with an 8-RHS
#     batch and time-to-tolerance, the full-size kernel table, and at
#     n = 2e6 the launch list of two iterations and ncu --set full of every
#     SpMV and wide-solve launch of the kernel table
set -e
R=${ROUND:-r01}
O=gpurun_out/prof
mkdir -p $O
PART=${PART:-all}

if [ "$PART" = all ] || [ "$PART" = c1 ]; then
SHORT="python bench.py --steps 3 --warmup 3 --no-tol --cpu-seconds 1 --batch 0"
python bench.py > $O/bench_$R.jsonl 2> $O/bench_$R.err
python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_reference_$R.jsonl 2> $O/bench_reference_$R.err
$SHORT > $O/short.jsonl 2> $O/short.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$R.csv $SHORT > $O/ncu_launch.log 2>&1
# the first timed iteration's 8 solves: 1 apply at start + 3 warm-up iterations precede it
ncu --set full --clock-control none --import-source on -k regex:k_trsv -s 32 -c 8 -o $O/trsv_$R -f $SHORT > $O/ncu_full.log 2>&1
ncu -i $O/trsv_$R.ncu-rep --page raw --csv > $O/trsv_$R.raw.csv
rm -f $O/trsv_$R.ncu-rep  # gpurun copies back at most 64 MiB
fi

if [ "$PART" = all ] || [ "$PART" = c4 ]; then
timeout 2400 python bench.py --config 4 --n 8000000 --blas-threads 64 --steps 20 --batch 8 --cpu-seconds 10 \
  > $O/bench_config4_n8m_$R.jsonl 2> $O/bench_config4_n8m_$R.err
timeout 1800 python scripts/kernel_table.py --n 8000000 > $O/kernel_table_config4_n8m_$R.json 2> $O/kernel_table_n8m.err
C4="python bench.py --config 4 --n 2000000 --blas-threads 64 --steps 2 --warmup 3 --no-tol --cpu-seconds 1 --batch 0"
$C4 > $O/c4_short.jsonl 2> $O/c4_short.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_config4_n2m_$R.csv $C4 > $O/ncu_c4_launch.log 2>&1
KT="python scripts/kernel_table.py --n 2000000 --reps 1"
$KT > $O/kernel_table_config4_n2m_$R.json 2> $O/kt2m.err
ncu --set full --clock-control none -k regex:"k_spmv|k_trsv_wide" -o $O/kt_$R -f $KT > $O/ncu_kt.log 2>&1
ncu -i $O/kt_$R.ncu-rep --page raw --csv > $O/kt_$R.raw.csv
rm -f $O/kt_$R.ncu-rep
fi
echo done
