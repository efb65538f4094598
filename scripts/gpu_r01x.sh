#!/bin/bash
# wide-solve prologue split (coalesced fill + level-0 pass): parity, config-4 kernel table at 8e6, bench at 2e6
O=gpurun_out/r01x
mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "wide or config or trsv or batch" > $O/pytest.log 2>&1; tail -2 $O/pytest.log
timeout 1500 python scripts/kernel_table.py --n 8000000 > $O/kernel_table_config4_n8m_r01.json 2> $O/kt8m.err
python -c "
import json; k=json.loads(open('$O/kernel_table_config4_n8m_r01.json').read().strip().splitlines()[-1]); print({a:b['ms'] for a,b in k['kernels'].items()})"
timeout 900 python bench.py --config 4 --n 2000000 --no-tol --batch 8 --steps 10 --cpu-seconds 1 --blas-threads 64 > $O/bench_c4_2m.jsonl 2> $O/bench_c4_2m.err
python -c "
import json; d=json.loads(open('$O/bench_c4_2m.jsonl').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['rhs_batch'])"
timeout 1500 python scripts/batch_conc.py --n 8000000 --batch 8 --iters 10 > $O/batch_conc_n8m.json 2> $O/batch_conc_n8m.err; tail -c 800 $O/batch_conc_n8m.json
