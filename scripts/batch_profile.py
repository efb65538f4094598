"""One batched (8-RHS) pcgls run on the configs[4] structure, for a kernel
launch list under ncu (experiments):

    ncu --metrics gpu__time_duration.sum --csv python scripts/batch_profile.py --n 8000000 --iters 2
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8_000_000)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--single", action="store_true", help="one RHS through pcgls instead")
    args = ap.parse_args()
    os.environ.setdefault("RSB_BLAS_THREADS", "64")
    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import workloads as W
    from paper_2603_28642_b200.ilup import ilup_factorize_cached

    A, B = W.config4(seed=4, n=args.n, nrhs=8)
    S, _ = P.column_scale(A)
    f = ilup_factorize_cached(S, P.IlupParams(p=10, tau=0.0, mu=1.0))
    pre = P.build_preconditioner(f, s_mode=P.SMode.INNER_CG)
    cfg = P.CglsConfig(norm_A=1.0, delta=1e-300, max_iters=args.iters)
    if args.single:
        x, rep = P.pcgls(S, B[0], pre, cfg)
    else:
        X, reps = P.pcgls_batch(S, B, pre, cfg)
    print("done")


if __name__ == "__main__":
    main()
