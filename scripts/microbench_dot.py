"""Device time of one exact-order dot (rsb_dot on device vectors) at several lengths:
a.b and the norm a.a (one operand stream).  RSB_BLAS_THREADS sets the dot order."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_28642_b200 import _lib as L
from paper_2603_28642_b200.device import DeviceBuffer, get_context
ctx = get_context(); out = {}; norm = {}
for n in (32768, 65536, 98304, 1 << 20, 8_000_000, 16_000_000):
    rng = np.random.default_rng(n); a = DeviceBuffer(ctx, n); b = DeviceBuffer(ctx, n)
    a.upload(rng.standard_normal(n)); b.upload(rng.standard_normal(n)); r = np.zeros(1); ts = []
    for k in range(13):
        ctx.mark(0); L.check(L.lib().rsb_dot(ctx.h, n, a.ptr, b.ptr, r.ctypes.data_as(L.f64p), L.RSB_DEVICE)); ctx.mark(1)
        if k >= 3: ts.append(ctx.elapsed_ms(0, 1))
    out[n] = round(1e3 * float(np.median(ts)), 2)
    ts = []
    for k in range(13):
        ctx.mark(0); L.check(L.lib().rsb_dot(ctx.h, n, a.ptr, a.ptr, r.ctypes.data_as(L.f64p), L.RSB_DEVICE)); ctx.mark(1)
        if k >= 3: ts.append(ctx.elapsed_ms(0, 1))
    norm[n] = round(1e3 * float(np.median(ts)), 2)
print(json.dumps({"blas_threads": os.environ.get("RSB_BLAS_THREADS", "1"), "dot_us": out, "norm_us": norm}))
