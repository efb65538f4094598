"""Time the wide triangular solves of the config-4 structure under several
analysis / launch settings (environment variables read when a matrix is
analysed or a solve launched), one ILUP, all in process, and check every
setting gives the same bits.

    python scripts/sweep_wide.py [--n 2000000] [--set NAME=ENV1=V1,ENV2=V2 ...]

Default settings: the current default, no within-level sort
(RSB_TRSV_SORT=0), register entries forced to 12 (RSB_WIDE_N=12), and the
level-synchronous kernel (RSB_TRSV_GRID=lsync).
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

DEFAULT_SETS = ["default=", "nosort=RSB_TRSV_SORT=0", "n12=RSB_WIDE_N=12", "n8=RSB_WIDE_N=8",
                "lsync=RSB_TRSV_GRID=lsync"]
KNOBS = ("RSB_TRSV_SORT", "RSB_WIDE_N", "RSB_TRSV_GRID", "RSB_WIDE_OCC", "RSB_WIDE_BACKOFF", "RSB_WIDE_P")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--set", nargs="*", default=DEFAULT_SETS)
    args = ap.parse_args()
    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import _lib as L
    from paper_2603_28642_b200 import workloads as W
    from paper_2603_28642_b200.device import DeviceBuffer, DeviceMatrix, get_context

    A, _ = W.config4(seed=4, n=args.n, nrhs=0)
    S, _ = P.column_scale(A)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=0.0, mu=1.0))
    ctx = get_context()
    n = f.U.ncols
    b = DeviceBuffer(ctx, n)
    b.upload(np.random.default_rng(0).standard_normal(n))
    x = DeviceBuffer(ctx, n)
    res, ref = {}, {}
    for spec in args.set:
        label, _, envs = spec.partition("=")
        for k in KNOBS:
            os.environ.pop(k, None)
        for kv in filter(None, envs.split(",")):
            k, v = kv.split("=", 1)
            os.environ[k] = v
        dL1, dU = DeviceMatrix(f.L1, ctx), DeviceMatrix(f.U, ctx)
        res[label] = {}
        for name, dm, kind in (("L1", dL1, L.TRI_LOWER_UNIT), ("L1T", dL1, L.TRI_LOWER_T_UNIT),
                               ("U", dU, L.TRI_UPPER)):
            ts = []
            for r in range(args.reps + 2):
                ctx.mark(0)
                L.check(L.lib().rsb_trsv(dm.h, kind, b.ptr, x.ptr, L.RSB_DEVICE))
                ctx.mark(1)
                if r >= 2:
                    ts.append(ctx.elapsed_ms(0, 1))
            out = x.download()
            if name in ref:
                assert np.array_equal(out, ref[name]), (label, name)
            ref.setdefault(name, out)
            res[label][name] = round(float(np.median(ts)), 4)
        res[label]["variant"] = {"L1": dL1.variant(L.TRI_LOWER_UNIT)[0], "U": dU.variant(L.TRI_UPPER)[0]}
        print(label, res[label], flush=True)
        del dL1, dU
    print(json.dumps(res))


if __name__ == "__main__":
    main()
