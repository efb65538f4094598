"""Device time and HBM rate of y = A x and z = A^T y on the config-4 structure.

    [RSB_SPMV=thread] python scripts/microbench_spmv.py [--n 8000000] [--reps 10]

Builds only A (no factorization): configs[4] structure at n unknowns, m = 2n
rows, column-scaled as the pipeline does.  Each launch is timed with CUDA
events on the context stream, L2 flushed before every launch (outside the
bracket).  Algorithmic bytes: 12 nnz + 4 (R + 1) + 8 C + 8 R
for an R x C product.  Prints one JSON line, including a checksum of the
outputs' bits so two kernel variants can be compared for identity.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8_000_000)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import _lib as L
    from paper_2603_28642_b200 import workloads as W
    from paper_2603_28642_b200.device import DeviceBuffer, DeviceMatrix, get_context

    t0 = time.perf_counter()
    A, _ = W.config4(seed=4, n=args.n, nrhs=0)
    A, _ = P.column_scale(A)
    t_gen = time.perf_counter() - t0
    ctx = get_context()
    m, n = A.nrows, A.ncols
    dm = DeviceMatrix(A, ctx)
    rng = np.random.default_rng(0)
    x = DeviceBuffer(ctx, n)
    x.upload(rng.standard_normal(n))
    yv = DeviceBuffer(ctx, m)
    yv.upload(rng.standard_normal(m))
    out_m = DeviceBuffer(ctx, m)
    out_n = DeviceBuffer(ctx, n)
    res = {"variant": os.environ.get("RSB_SPMV", "tile"), "n": n, "m": m, "nnz": int(A.nnz),
           "generate_s": round(t_gen, 1)}
    digest = hashlib.sha256()
    for name, fn, src, dst, R, C in (("A_x", L.lib().rsb_matvec, x, out_m, m, n),
                                     ("At_y", L.lib().rsb_matvec_transpose, yv, out_n, n, m)):
        ts = []
        for r in range(args.reps + 2):
            L.check(L.lib().rsb_l2_flush(ctx.h))
            ctx.mark(0)
            L.check(fn(dm.h, src.ptr, dst.ptr, L.RSB_DEVICE))
            ctx.mark(1)
            if r >= 2:
                ts.append(ctx.elapsed_ms(0, 1))
        ms = float(np.median(ts))
        nbytes = 12 * A.nnz + 4 * (R + 1) + 8 * C + 8 * R
        res[name] = {"ms": round(ms, 4), "GBps": round(nbytes / (ms / 1e3) / 1e9, 1),
                     "alg_bytes": int(nbytes)}
        digest.update(dst.download().tobytes())
    res["checksum"] = digest.hexdigest()[:16]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
