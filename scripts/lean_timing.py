"""Segment-wait vs level-run cycles of the lean triangular solve on config 1
(RSB_TRSV_PROFILE=1: thread 0 accumulates clock64 phases)."""
import ctypes, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["RSB_TRSV_PROFILE"] = "1"
import paper_2603_28642_b200 as P
from paper_2603_28642_b200 import _lib as L
from paper_2603_28642_b200 import workloads as W
from paper_2603_28642_b200.device import DeviceBuffer, DeviceMatrix, get_context
A, _ = W.config1(seed=1, g=256)
S, _ = P.column_scale(A)
f = P.ilup_factorize(S, P.IlupParams(p=10, tau=0.0, mu=1.0))
ctx = get_context(); n = f.U.ncols
b = DeviceBuffer(ctx, n); b.upload(np.random.default_rng(0).standard_normal(n)); x = DeviceBuffer(ctx, n)
L.lib().rsb_trsv_profile.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_longlong)]
out = {}
for name, M, kind in (("L1", f.L1, L.TRI_LOWER_UNIT), ("L1T", f.L1, L.TRI_LOWER_T_UNIT), ("U", f.U, L.TRI_UPPER)):
    dm = DeviceMatrix(M, ctx)
    for _ in range(3):
        L.check(L.lib().rsb_trsv(dm.h, kind, b.ptr, x.ptr, L.RSB_DEVICE))
    c = (ctypes.c_longlong * 8)()
    L.check(L.lib().rsb_trsv_profile(dm.h, kind, c))
    nl, ns = c[5], max(c[2], 1)
    out[name] = {"cycles_per_level": round(c[1] / nl, 1), 
                 "producer_chunk_wait_per_level": round(c[6] / nl, 1),
                 "prologue_cycles": c[7], "loop_cycles": c[1], "levels": nl, "chunks": c[4]}
print(json.dumps(out))
