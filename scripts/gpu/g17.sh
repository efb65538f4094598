mkdir -p gpurun_out
export RSB_FACTOR_CACHE=/tmp/rsb_fc
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/g17_pytest.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/g17_pytest.log
timeout 1500 python bench.py --no-tol > gpurun_out/g17_b8m.log 2>&1; echo b8m rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/g17_b8m.log').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step')}, d['e2e']['value'], d['roofline']['achieved'], d['roofline']['share_of_step'], d['parity'], d['rhs_batch']['device']['value'])
PY
