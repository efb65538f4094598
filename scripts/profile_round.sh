#!/bin/bash
# Measurement pass for profiles/ (run on the GPU box through gpurun, from the
# repo root):  bench lines, the ncu launch list of a short bench run, and one
# `ncu --set full` capture of the triangular solves of one timed iteration.
# Each ncu command runs only after the same command exited 0 without ncu.
# Outputs go to gpurun_out/prof/; scripts/summarize_profiles.py turns them
# into the profiles/ files.
set -e
R=${ROUND:-r01}
O=gpurun_out/prof
mkdir -p $O
SHORT="python bench.py --steps 3 --warmup 3 --no-tol --cpu-seconds 1 --batch 0"
python bench.py > $O/bench_$R.jsonl 2> $O/bench_$R.err
python bench.py --impl reference --steps 10 --warmup 3 > $O/bench_reference_$R.jsonl 2> $O/bench_reference_$R.err
$SHORT > $O/short.jsonl 2> $O/short.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_$R.csv $SHORT > $O/ncu_launch.log 2>&1
# the first timed iteration's 8 solves: 1 apply at start + 3 warm-up iterations precede it
ncu --set full --clock-control none --import-source on -k regex:k_trsv -s 32 -c 8 -o $O/trsv_$R -f $SHORT > $O/ncu_full.log 2>&1
ncu -i $O/trsv_$R.ncu-rep --page raw --csv > $O/trsv_$R.raw.csv
echo done
