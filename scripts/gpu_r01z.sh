#!/bin/bash
# final state: full GPU suite, smoke, default bench line
O=gpurun_out/r01z
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo pytest=$? >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 600 python bench.py > $O/bench.jsonl 2> $O/bench.err
python -c "
import json; d=json.loads(open('$O/bench.jsonl').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['rhs_batch']['value'], d['gpu_launches'])"
