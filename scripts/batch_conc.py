"""RHS-iterations/s of pcgls_batch at several concurrency caps (RSB_BATCH_CONC).

    python scripts/batch_conc.py [--config 4] [--n 2000000] [--batch 8] [--iters 10]

One factorization, then pcgls_batch over the same B with 1, 2, 4 and `batch`
solves iterating at once; prints one JSON line.  The results of every cap are
checked bit-identical to the first.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--blas-threads", type=int, default=64)
    a = ap.parse_args()
    import bench
    import paper_2603_28642_b200 as P

    sys.argv = [sys.argv[0], "--config", str(a.config), "--n", str(a.n), "--blas-threads", str(a.blas_threads)]
    args = bench.parse()
    os.environ["RSB_BLAS_THREADS"] = str(a.blas_threads)
    A, b, st, name, _ = bench.make_workload(args, 0)
    S, f, pre, mode, times = bench.setup(args, A, st)
    norm_a = P.power_method_norm2(S, 100)
    rng = np.random.default_rng(77)
    B = np.stack([b] + [b + 1e-3 * rng.standard_normal(len(b)) for _ in range(a.batch - 1)])
    cfg = P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=a.iters)
    out = {"workload": name, "batch": a.batch, "iters": a.iters, "ilup_s": round(times["ilup_host_s"], 1)}
    ref = None
    for conc in sorted({1, 2, 4, a.batch}):
        os.environ["RSB_BATCH_CONC"] = str(conc)
        P.pcgls_batch(S, B, pre, P.CglsConfig(norm_A=norm_a, delta=1e-300, max_iters=2))
        t0 = time.perf_counter()
        X, reps = P.pcgls_batch(S, B, pre, cfg)
        dt = time.perf_counter() - t0
        its = sum(r.its for r in reps)
        if ref is None:
            ref = X
        out[f"conc{conc}"] = {"rhs_iter_per_s": round(its / dt, 2), "seconds": round(dt, 3),
                              "identical": bool(np.array_equal(np.asarray(X), np.asarray(ref)))}
    os.environ.pop("RSB_BATCH_CONC")
    t0 = time.perf_counter()
    X, reps = P.pcgls_batch(S, B, pre, cfg)
    dt = time.perf_counter() - t0
    out["default"] = {"rhs_iter_per_s": round(sum(r.its for r in reps) / dt, 2), "seconds": round(dt, 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
