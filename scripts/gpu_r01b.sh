#!/bin/bash
# one gpurun pass: GPU tests, SpMV microbench both variants + ncu, dot microbench
O=gpurun_out/r01b
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
python scripts/microbench_spmv.py --n 2000000 > $O/spmv_tile_2m.json 2>&1
RSB_SPMV=thread python scripts/microbench_spmv.py --n 2000000 > $O/spmv_thread_2m.json 2>&1
cat $O/spmv_*.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 4 -c 4 -o $O/spmv_tile -f python scripts/microbench_spmv.py --n 2000000 --reps 1 > $O/ncu_tile.log 2>&1
RSB_SPMV=thread timeout 600 ncu --set full --clock-control none -k regex:k_spmv -s 4 -c 4 -o $O/spmv_thread -f python scripts/microbench_spmv.py --n 2000000 --reps 1 > $O/ncu_thread.log 2>&1
for t in 1 8 64; do RSB_BLAS_THREADS=$t python scripts/microbench_dot.py > $O/dot_t$t.json 2>&1; done
cat $O/dot_t*.json
