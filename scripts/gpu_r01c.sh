#!/bin/bash
O=gpurun_out/r01c
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python scripts/microbench_spmv.py --n 2000000 > $O/spmv_tile_2m.json 2>&1
RSB_SPMV=thread python scripts/microbench_spmv.py --n 2000000 > $O/spmv_thread_2m.json 2>&1
cat $O/spmv_*.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 2 -c 2 -o $O/spmv_tile -f python scripts/microbench_spmv.py --n 2000000 --reps 1 > $O/ncu_tile.log 2>&1
RSB_SPMV=thread timeout 600 ncu --set full --clock-control none -k regex:k_spmv -s 2 -c 1 -o $O/spmv_thread -f python scripts/microbench_spmv.py --n 2000000 --reps 1 > $O/ncu_thread.log 2>&1
timeout 900 python scripts/microbench_trsv.py --config 4 --n 2000000 > $O/trsv_lsync_2m.json 2>&1
RSB_TRSV_GRID=syncfree timeout 900 python scripts/microbench_trsv.py --config 4 --n 2000000 > $O/trsv_syncfree_2m.json 2>&1
cat $O/trsv_*.json
timeout 1200 python bench.py --config 4 --n 2000000 --no-tol --batch 0 --steps 10 --cpu-seconds 5 --blas-threads 64 > $O/bench_c4_2m_t64.jsonl 2> $O/bench_c4_2m_t64.err
tail -c 600 $O/bench_c4_2m_t64.jsonl
