"""Per-kernel device time and HBM rate of every kernel class of a pcgls
iteration on the configs[4] structure (SURVEY.md 8(d) roofline table).

    python scripts/kernel_table.py [--n 8000000] [--mu 1.0] [--reps 5] [--blas-threads 64]

Builds the config-4 problem at n unknowns (generate, column_scale, ILUP on
the host), uploads A and the factors, and times each kernel class alone
with CUDA events on the context stream, L2 flushed before every launch
(outside the bracket): A x (CSR), A^T y (CSC), L2 t (CSR), L2^T w (CSC),
the three triangular solves of the apply (L1, L1^T, U; their level counts),
and the exact-order dots of length m, n and s.  Algorithmic bytes follow
SURVEY.md 8(d): SpMV 12 N + 4 (R + 1) + 8 C + 8 R; triangular solve
12 N + 4 (n + 1) + 16 n; dot 16 len.  Prints one JSON line; the peak is
MEASURED_PEAKS.json's hbm_gbs.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, HERE)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8_000_000)
    ap.add_argument("--mu", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--blas-threads", type=int, default=64)
    args = ap.parse_args()
    os.environ["RSB_BLAS_THREADS"] = str(args.blas_threads)
    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import _lib as L
    from paper_2603_28642_b200 import workloads as W
    from paper_2603_28642_b200.device import DeviceBuffer, DeviceMatrix, get_context

    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as fh:
            peak = float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        peak = 6650.0
    t0 = time.perf_counter()
    A, _ = W.config4(seed=4, n=args.n, nrhs=0)
    S, _ = P.column_scale(A)
    t_gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    from paper_2603_28642_b200.ilup import ilup_factorize_cached

    f = ilup_factorize_cached(S, P.IlupParams(p=10, tau=0.0, mu=args.mu))  # $RSB_FACTOR_CACHE
    t_ilup = time.perf_counter() - t0
    ctx = get_context()
    m, n, s = S.nrows, S.ncols, f.L2.nrows
    rng = np.random.default_rng(0)

    def buf(k):
        b = DeviceBuffer(ctx, k)
        b.upload(rng.standard_normal(k))
        return b

    vm, vn, vs, om, on, os_ = buf(m), buf(n), buf(s), buf(m), buf(n), buf(s)

    def timed(fn):
        ts = []
        for r in range(args.reps + 2):
            L.check(L.lib().rsb_l2_flush(ctx.h))
            ctx.mark(0)
            L.check(fn())
            ctx.mark(1)
            if r >= 2:
                ts.append(ctx.elapsed_ms(0, 1))
        return float(np.median(ts))

    rows = {}

    def record(name, ms, nbytes, **extra):
        gbs = nbytes / (ms / 1e3) / 1e9
        rows[name] = dict(ms=round(ms, 4), alg_bytes=int(nbytes), GBps=round(gbs, 1), frac=round(gbs / peak, 4),
                          **extra)

    dA = DeviceMatrix(S, ctx)
    dL2 = DeviceMatrix(f.L2, ctx)
    lib = L.lib()
    spmv = lambda N, R, C: 12 * N + 4 * (R + 1) + 8 * C + 8 * R  # noqa: E731
    record("A_x (CSR)", timed(lambda: lib.rsb_matvec(dA.h, vn.ptr, om.ptr, L.RSB_DEVICE)), spmv(S.nnz, m, n))
    record("A^T_y (CSC)", timed(lambda: lib.rsb_matvec_transpose(dA.h, vm.ptr, on.ptr, L.RSB_DEVICE)),
           spmv(S.nnz, n, m))
    record("L2_t (CSR)", timed(lambda: lib.rsb_matvec(dL2.h, vn.ptr, os_.ptr, L.RSB_DEVICE)), spmv(f.L2.nnz, s, n))
    record("L2^T_w (CSC)", timed(lambda: lib.rsb_matvec_transpose(dL2.h, vs.ptr, on.ptr, L.RSB_DEVICE)),
           spmv(f.L2.nnz, n, s))
    tri = lambda N: 12 * N + 4 * (n + 1) + 16 * n  # noqa: E731
    for name, M, kind in (("L1 solve", f.L1, L.TRI_LOWER_UNIT), ("L1^T solve", f.L1, L.TRI_LOWER_T_UNIT),
                          ("U solve", f.U, L.TRI_UPPER)):
        dm = dA if M is S else DeviceMatrix(M, ctx)
        lv = dm.levels(kind)
        var = dm.variant(kind)[0]
        ms = timed(lambda: lib.rsb_trsv(dm.h, kind, vn.ptr, on.ptr, L.RSB_DEVICE))
        record(name, ms, tri(M.nnz), levels=lv[0], max_width=lv[1], variant=var, us_per_level=round(1e3 * ms / lv[0], 2))
    out = np.zeros(1)
    for name, k, a in (("dot m", m, vm), ("dot n", n, vn), ("dot s", s, vs)):
        record(f"{name} (T={args.blas_threads})",
               timed(lambda: lib.rsb_dot(ctx.h, k, a.ptr, a.ptr, out.ctypes.data_as(L.f64p), L.RSB_DEVICE)), 16 * k)
    print(json.dumps({"config": f"configs[4] structure n={n} m={m} s={s} mu={args.mu}",
                      "nnz": {"A": int(S.nnz), "L1": int(f.L1.nnz), "L2": int(f.L2.nnz), "U": int(f.U.nnz)},
                      "peak_GBps": peak, "generate_s": round(t_gen, 1), "ilup_s": round(t_ilup, 1),
                      "kernels": rows}))


if __name__ == "__main__":
    main()
