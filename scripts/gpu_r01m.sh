#!/bin/bash
O=gpurun_out/r01o
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 900 python scripts/sweep_wide.py --n 2000000 --set default= > $O/sweep.log 2>&1; tail -4 $O/sweep.log
timeout 1200 python bench.py --config 4 --n 2000000 --no-tol --batch 0 --steps 10 --cpu-seconds 3 --blas-threads 64 > $O/bench_c4_2m_t64.jsonl 2> $O/bench_c4_2m_t64.err
python -c "
import json; d=json.loads(open('$O/bench_c4_2m_t64.jsonl').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['share_of_step'], d['e2e']['value'])"
