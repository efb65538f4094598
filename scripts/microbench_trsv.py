"""Time each triangular solve of the config-1 preconditioner on the device.

    RSB_TRSV_VARIANT=cta|grid python scripts/microbench_trsv.py [--grid 256] [--mu 1.0]

Prints one JSON line: per kind (L1 forward, L1^T, U backward) the device ms
per solve (CUDA events, median of repeats), levels, and GB/s of the
algorithmic bytes (12 nnz + 20 n + 4).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--mu", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--n", type=int, default=1_000_000)
    args = ap.parse_args()
    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import _lib as L
    from paper_2603_28642_b200 import workloads as W
    from paper_2603_28642_b200.device import DeviceBuffer, DeviceMatrix, get_context

    if args.config == 4:
        A, _ = W.config4(seed=4, n=args.n, nrhs=1)
    else:
        A, _ = W.config1(seed=1, g=args.grid)
    S, _ = P.column_scale(A)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=0.0, mu=args.mu))
    ctx = get_context()
    n = f.U.ncols
    rng = np.random.default_rng(0)
    b = DeviceBuffer(ctx, n)
    b.upload(rng.standard_normal(n))
    x = DeviceBuffer(ctx, n)
    out = {"variant": os.environ.get("RSB_TRSV_VARIANT", "auto"), "n": n, "mu": args.mu}
    for name, M, kind in (("L1", f.L1, L.TRI_LOWER_UNIT), ("L1T", f.L1, L.TRI_LOWER_T_UNIT),
                          ("U", f.U, L.TRI_UPPER)):
        dm = DeviceMatrix(M, ctx)
        lv = dm.levels(kind)
        ts = []
        for r in range(args.reps + 3):
            ctx.mark(0)
            L.check(L.lib().rsb_trsv(dm.h, kind, b.ptr, x.ptr, L.RSB_DEVICE))
            ctx.mark(1)
            if r >= 3:
                ts.append(ctx.elapsed_ms(0, 1))
        ms = float(np.median(ts))
        nbytes = 12 * M.nnz + 20 * n + 4
        out[name] = {"ms": ms, "levels": lv[0], "max_width": lv[1], "nnz": M.nnz,
                     "us_per_level": 1e3 * ms / lv[0], "GBps": nbytes / (ms / 1e3) / 1e9}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
