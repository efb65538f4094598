#!/bin/bash
# SpMV thread-per-row register batches: A x / A^T y at config-4 size, variants, parity
O=gpurun_out/${OUT:-r01s}
mkdir -p $O
timeout 600 python scripts/microbench_spmv.py --n 8000000 > $O/spmv_auto.json 2> $O/spmv_auto.err; cat $O/spmv_auto.json
RSB_SPMV=tile timeout 600 python scripts/microbench_spmv.py --n 8000000 > $O/spmv_tile.json 2> $O/spmv_tile.err; cat $O/spmv_tile.json
timeout 900 python -m pytest tests -m gpu -x -q -k "spmv or matvec or config" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
