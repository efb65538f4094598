#!/bin/bash
# config 4 at full size after the wide-prologue split and the batch concurrency cap
O=gpurun_out/prof
mkdir -p $O
timeout 2400 python bench.py --config 4 --n 8000000 --blas-threads 64 --steps 20 --batch 8 --cpu-seconds 10 \
  > $O/bench_config4_n8m_r01.jsonl 2> $O/bench_config4_n8m_r01.err
python -c "
import json; d=json.loads(open('$O/bench_config4_n8m_r01.jsonl').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['rhs_batch']['value'], d['time_to_tol'])"
