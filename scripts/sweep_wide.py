"""Sweep the sync-free wide solve's resident blocks per SM and back-off cap
(RSB_WIDE_OCC, RSB_WIDE_BACKOFF) on the config-4 structure; also the
level-synchronous variant.  One ILUP, all variants timed in process.

    python scripts/sweep_wide.py [--n 2000000]
"""
import argparse, json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--reps", type=int, default=7)
    ap.add_argument("--quick", action="store_true", help="default settings only")
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
    b = DeviceBuffer(ctx, n); b.upload(np.random.default_rng(0).standard_normal(n))
    x = DeviceBuffer(ctx, n)
    res = {}
    for grid in ("syncfree", "lsync"):
        os.environ["RSB_TRSV_GRID"] = grid
        mats = {"L1": (DeviceMatrix(f.L1, ctx), L.TRI_LOWER_UNIT), "L1T": (None, L.TRI_LOWER_T_UNIT),
                "U": (DeviceMatrix(f.U, ctx), L.TRI_UPPER)}
        mats["L1T"] = (mats["L1"][0], L.TRI_LOWER_T_UNIT)
        settings = [(o, bo) for o in (1, 2, 3) for bo in (128, 512, 2048)] if grid == "syncfree" else [(0, 0)]
        if args.quick:
            settings = [(3, 128)] if grid == "syncfree" else [(0, 0)]
        ref = {}
        for occ, bo in settings:
            if occ:
                os.environ["RSB_WIDE_OCC"], os.environ["RSB_WIDE_BACKOFF"] = str(occ), str(bo)
            key = f"{grid} occ={occ} backoff={bo}"
            res[key] = {}
            for name, (dm, kind) in mats.items():
                ts = []
                for r in range(args.reps + 2):
                    ctx.mark(0)
                    L.check(L.lib().rsb_trsv(dm.h, kind, b.ptr, x.ptr, L.RSB_DEVICE))
                    ctx.mark(1)
                    if r >= 2:
                        ts.append(ctx.elapsed_ms(0, 1))
                out = x.download()
                if name in ref:
                    assert np.array_equal(out, ref[name]), key
                ref.setdefault(name, out)
                res[key][name] = round(float(np.median(ts)), 4)
            print(key, res[key], flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
