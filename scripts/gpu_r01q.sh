#!/bin/bash
# lean-solve prologue: per-solve event time, loop vs prologue cycles, bench
O=gpurun_out/${OUT:-r01q}
mkdir -p $O
timeout 300 python scripts/lean_timing.py > $O/lean_timing.json 2> $O/lean_timing.err; cat $O/lean_timing.json
timeout 300 python scripts/microbench_trsv.py > $O/trsv.json 2> $O/trsv.err; cat $O/trsv.json
timeout 600 python -m pytest tests -m gpu -x -q > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 600 python bench.py --no-tol --cpu-seconds 2 > $O/bench.jsonl 2> $O/bench.err
python -c "
import json; d=json.loads(open('$O/bench.jsonl').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['share_of_step'])"
