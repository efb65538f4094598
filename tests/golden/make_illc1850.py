"""Golden fixture for the reference's bundled paper matrix illc1850 (the
robust parity gate of SURVEY.md §0/§8(c); acceptance band at
pkg/tests/test_acceptance.py:155-175, paper Table 3 row 19).

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_illc1850.py

Runs the REFERENCE package in this container, with the settings of its own
acceptance test (solve_pipeline, test_acceptance.py:44-52): Matrix Market
read, column_scale, ILUP(p=10, tau=0, mu=0.1), power_method_norm2(100,
seed 42), b = default_rng(42).uniform(-1, 1, m), delta 1e-10, 2000
iterations, in the dense, cg(2) and identity coupling modes.  Stores the
scaled matrix, b, norm_A, the factors, and per mode x, the SolveReport and
one preconditioner application, in tests/golden/illc1850.npz + .json.  The
GPU box has no reference: tests/test_gpu_illc1850.py checks the device path
against these outputs.
"""

from __future__ import annotations

import json
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

import rowsplit as rs  # noqa: E402

MTX = "/root/reference/pkg/data/illc1850.mtx"


def csc(prefix, M):
    return {f"{prefix}_shape": np.array([M.nrows, M.ncols]), f"{prefix}_ptr": M.col_ptr,
            f"{prefix}_idx": M.row_idx, f"{prefix}_val": M.values}


def main():
    A, info = rs.read_matrix_market_ex(MTX)
    S, sc = rs.column_scale(A)
    f = rs.ilup_factorize(S, rs.IlupParams(p=10, tau=0.0, mu=0.1, small=1e-10))
    rng = np.random.default_rng(42)
    b = rng.uniform(-1.0, 1.0, S.nrows)
    norm_a = rs.power_method_norm2(S, iters=100, seed=42)
    out = {"b": b, "norm_A": np.array([norm_a]), "perm": f.row_perm.perm, "nmod": np.array([f.nmod]),
           "row_counts": f.row_counts_final}
    out.update(csc("S", S))
    for k in ("L1", "L2", "U"):
        out.update(csc(k, getattr(f, k)))
    meta = {"matrix": "illc1850 (pkg/data/illc1850.mtx)", "shape": [S.nrows, S.ncols], "nnz": int(S.nnz),
            "params": {"p": 10, "tau": 0.0, "mu": 0.1, "small": 1e-10}, "delta": 1e-10, "max_iters": 2000,
            "seed": 42, "reports": {}}
    arng = np.random.default_rng(7)
    n = S.ncols
    r1, r2 = arng.standard_normal(n), arng.standard_normal(S.nrows - n)
    out["r1"], out["r2"] = r1, r2
    for mode in ("dense", "cg", "identity"):
        pre = rs.build_preconditioner(f, s_mode=rs.SMode(mode), cg_iters=2)
        cfg = rs.CglsConfig(norm_A=norm_a, delta=1e-10, max_iters=2000, estimator_delay=5)
        x, rep = rs.pcgls(S, b, pre, cfg)
        out[f"x_{mode}"] = x
        out[f"h_{mode}"] = pre.apply(r1, r2)
        meta["reports"][mode] = rep.to_dict()
    np.savez_compressed(os.path.join(HERE, "illc1850.npz"), **out)
    with open(os.path.join(HERE, "illc1850.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print({m: (r["its"], r["converged"]) for m, r in meta["reports"].items()})


if __name__ == "__main__":
    main()
