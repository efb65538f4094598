#!/bin/bash
O=gpurun_out/r01j
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python bench.py --steps 30 --no-tol --batch 0 --cpu-seconds 2 > $O/bench_c1.jsonl 2> $O/bench_c1.err
timeout 1200 python bench.py --config 4 --n 2000000 --no-tol --batch 0 --steps 10 --cpu-seconds 3 --blas-threads 64 > $O/bench_c4_2m_t64.jsonl 2> $O/bench_c4_2m_t64.err
for f in $O/bench_*.jsonl; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['roofline']['share_of_step'], d['e2e']['value'])"; done
