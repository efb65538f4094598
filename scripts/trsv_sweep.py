"""Triangular-solve variants on the configs[4] structure (experiments).

    python scripts/trsv_sweep.py [--n 8000000] [--reps 5] [--ls-p 1,2,4] [--syncfree]

Times the three solves of the apply (L1, L1^T, U) alone, L2 flushed before
each launch, for the level-synchronous kernel at several items-in-flight
settings (RSB_LS_P) and optionally the sync-free kernel; checks every
variant's output against the first one bit for bit.  One JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8_000_000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--ls-p", default="1,2,4")
    ap.add_argument("--syncfree", action="store_true")
    ap.add_argument("--occ", default="", help="comma list of RSB_LS_OCC caps to sweep too")
    ap.add_argument("--env", action="append", default=[],
                    help="extra sync-free settings, e.g. --env RSB_TRSV_EVICT=1 (repeatable; ';' joins several)")
    args = ap.parse_args()
    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import _lib as L
    from paper_2603_28642_b200 import workloads as W
    from paper_2603_28642_b200.device import DeviceBuffer, DeviceMatrix, get_context
    from paper_2603_28642_b200.ilup import ilup_factorize_cached

    A, _ = W.config4(seed=4, n=args.n, nrhs=0)
    S, _ = P.column_scale(A)
    f = ilup_factorize_cached(S, P.IlupParams(p=10, tau=0.0, mu=1.0))
    ctx = get_context()
    n = f.U.ncols
    rng = np.random.default_rng(0)
    b = DeviceBuffer(ctx, n)
    b.upload(rng.standard_normal(n))
    x = DeviceBuffer(ctx, n)
    lib = L.lib()
    tri = lambda N: 12 * N + 4 * (n + 1) + 16 * n  # noqa: E731

    def timed(fn):
        ts = []
        for r in range(args.reps + 2):
            L.check(lib.rsb_l2_flush(ctx.h))
            ctx.mark(0)
            L.check(fn())
            ctx.mark(1)
            if r >= 2:
                ts.append(ctx.elapsed_ms(0, 1))
        return float(np.median(ts))

    out = {}
    ref = {}
    settings = [("ls", p, o) for p in args.ls_p.split(",") for o in ([""] + [v for v in args.occ.split(",") if v])]
    if args.syncfree:
        settings.append(("syncfree", "", ""))
    for e in args.env:
        settings.append(("syncfree+" + e, "", ""))
    for fam, p, occ in settings:
        key = f"{fam}" + (f"_P{p}" if p else "") + (f"_occ{occ}" if occ else "")
        for e in [v for a in args.env for v in a.split(";")]:
            os.environ.pop(e.split("=")[0], None)
        os.environ["RSB_TRSV_GRID"] = "syncfree" if fam.startswith("syncfree") else "levelsync"
        if fam.startswith("syncfree+"):
            for e in fam.split("+", 1)[1].split(";"):
                k_, v_ = e.split("=")
                os.environ[k_] = v_
        os.environ["RSB_LS_P"] = p or "4"
        if occ:
            os.environ["RSB_LS_OCC"] = occ
        else:
            os.environ.pop("RSB_LS_OCC", None)
        row = {}
        for name, M, kind in (("L1", f.L1, L.TRI_LOWER_UNIT), ("L1T", f.L1, L.TRI_LOWER_T_UNIT),
                              ("U", f.U, L.TRI_UPPER)):
            Mc = P.CscMatrix(M.nrows, M.ncols, M.col_ptr, M.row_idx, M.values)
            dm = DeviceMatrix(Mc, ctx)
            ms = timed(lambda: lib.rsb_trsv(dm.h, kind, b.ptr, x.ptr, L.RSB_DEVICE))
            got = x.download()
            if name not in ref:
                ref[name] = got
            same = bool(np.array_equal(got.view(np.int64), ref[name].view(np.int64)))
            gbs = tri(M.nnz) / (ms / 1e3) / 1e9
            row[name] = {"ms": round(ms, 4), "GBps": round(gbs, 1), "bitwise_vs_first": same,
                         "variant": dm.variant(kind)[0]}
            del dm
        out[key] = row
    print(json.dumps({"n": n, "nnz": {"L1": int(f.L1.nnz), "U": int(f.U.nnz)}, "results": out}))


if __name__ == "__main__":
    main()
