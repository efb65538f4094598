#!/bin/bash
# SpMV staging in rounds of 8: A x (thread / tile), A^T y at 8e6; kernel table at 2e6 (L2 products); parity
O=gpurun_out/${OUT:-r01u}
mkdir -p $O
timeout 600 python scripts/microbench_spmv.py --n 8000000 > $O/spmv_auto.json 2> $O/spmv_auto.err; cat $O/spmv_auto.json
RSB_SPMV=tile timeout 600 python scripts/microbench_spmv.py --n 8000000 > $O/spmv_tile.json 2> $O/spmv_tile.err; cat $O/spmv_tile.json
timeout 900 python -m pytest tests -m gpu -x -q -k "spmv or matvec or config or kernel" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 1200 python scripts/kernel_table.py --n 2000000 --reps 5 > $O/kt2m.json 2> $O/kt2m.err; head -c 1500 $O/kt2m.json
