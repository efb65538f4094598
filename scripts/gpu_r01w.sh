#!/bin/bash
# final round check: full GPU suite + smoke, then the config-1 profiling pass
O=gpurun_out/r01w
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
PART=c1 timeout 1500 bash scripts/profile_round.sh
timeout 900 python scripts/batch_conc.py --n 2000000 --batch 8 --iters 10 > $O/batch_conc.json 2> $O/batch_conc.err; tail -c 800 $O/batch_conc.json
