#!/bin/bash
O=gpurun_out/r01g
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 1500 python scripts/kernel_table.py --n 8000000 > $O/kernel_table_8m.json 2> $O/kernel_table_8m.err
cat $O/kernel_table_8m.json
timeout 1800 python bench.py --config 4 --n 8000000 --no-tol --batch 0 --steps 10 --cpu-seconds 10 --blas-threads 64 > $O/bench_c4_8m_t64.jsonl 2> $O/bench_c4_8m_t64.err
tail -c 400 $O/bench_c4_8m_t64.jsonl
