#!/bin/bash
# lean-solve experiment: cycles per level + the lean parity tests + bench
O=gpurun_out/${OUT:-r01t}
mkdir -p $O
timeout 300 python scripts/lean_timing.py > $O/lean_timing.json 2> $O/lean_timing.err; cat $O/lean_timing.json
timeout 900 python -m pytest tests -m gpu -x -q -k "${TK:-lean or trsv or tri}" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 600 python bench.py --no-tol --cpu-seconds 1 --batch 0 > $O/bench.jsonl 2> $O/bench.err
python -c "
import json; d=json.loads(open('$O/bench.jsonl').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'])"
