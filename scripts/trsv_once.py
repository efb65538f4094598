"""One of each triangular solve of the cg(2) apply (L1, L1^T, U) on the
configs[4] structure, for an ncu capture (the bench's roofline `traffic`):

    ncu --set full -k regex:"k_trsv|k_wide|k_fill" python scripts/trsv_once.py --n 8000000

Each kind runs twice; the second run of each is the measured one (the
first pays the analysis)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8_000_000)
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
    b = DeviceBuffer(ctx, n)
    b.upload(np.random.default_rng(0).standard_normal(n))
    x = DeviceBuffer(ctx, n)
    dL1, dU = DeviceMatrix(f.L1, ctx), DeviceMatrix(f.U, ctx)
    for dm, kind in ((dL1, L.TRI_LOWER_UNIT), (dL1, L.TRI_LOWER_T_UNIT), (dU, L.TRI_UPPER)):
        for _ in range(2):
            L.check(L.lib().rsb_l2_flush(ctx.h))
            L.check(L.lib().rsb_trsv(dm.h, kind, b.ptr, x.ptr, L.RSB_DEVICE))
    ctx.sync()
    print("done")


if __name__ == "__main__":
    main()
