"""Host setup / upload / analysis phase timings on the configs[4] structure (experiments)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RSB_DEBUG_ANALYSIS"] = "1"
import paper_2603_28642_b200 as P  # noqa: E402
from paper_2603_28642_b200 import device as D  # noqa: E402
from paper_2603_28642_b200 import workloads as W  # noqa: E402
from paper_2603_28642_b200.ilup import ilup_factorize_cached  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8_000_000
A, _ = W.config4(seed=4, n=n, nrhs=0)
S, _ = P.column_scale(A)
f = ilup_factorize_cached(S, P.IlupParams(p=10, tau=0.0, mu=1.0))
pre = P.build_preconditioner(f, s_mode=P.SMode.INNER_CG)
ctx = D.get_context()
t0 = time.perf_counter()
dA = D.device_matrix(S, ctx)
ctx.sync()
print("upload A", time.perf_counter() - t0, flush=True)
t0 = time.perf_counter()
dpre = D.device_preconditioner(pre, ctx)
ctx.sync()
print("upload + analyse preconditioner", time.perf_counter() - t0, flush=True)
