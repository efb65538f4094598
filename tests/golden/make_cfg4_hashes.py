"""Pin full-size host setup to the REFERENCE: run the reference package's
column_scale + ilup_factorize (pkg/src/rowsplit/sparse_core.py:405-425,
ilup.py:211-368) on the config-4 structure and record SHA-256 digests of
every output array, so the GPU box (which has no reference) can check that
the native ILUP produced the reference's factors bit for bit.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_cfg4_hashes.py 100000 8000000

Writes tests/golden/cfg4_factor_hashes.json (one entry per n).  The
reference ILUP at mu = 1 is linear on this structure (~0.5 ms/column), so
n = 8e6 takes over an hour; it runs once, here, in the build container.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

OUT = os.path.join(HERE, "cfg4_factor_hashes.json")


def digest(a):
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.tobytes()).hexdigest() + f":{a.dtype.str}:{a.size}"


def factor_digests(S_values, scale, f):
    d = {"S_values": digest(S_values), "scale": digest(scale), "perm": digest(f.row_perm.perm),
         "nmod": int(f.nmod), "row_counts": digest(f.row_counts_final)}
    for k in ("L1", "L2", "U"):
        M = getattr(f, k)
        d[k] = {"shape": [int(M.nrows), int(M.ncols)], "nnz": int(M.nnz), "ptr": digest(M.col_ptr),
                "idx": digest(M.row_idx), "val": digest(M.values)}
    return d


def main(ns):
    import rowsplit as rs

    from paper_2603_28642_b200 import workloads as W

    try:
        with open(OUT) as fh:
            table = json.load(fh)
    except OSError:
        table = {}
    for n in ns:
        t0 = time.perf_counter()
        A, _ = W.config4(seed=4, n=n, nrhs=0)
        Ar = rs.CscMatrix(A.nrows, A.ncols, A.col_ptr, A.row_idx, A.values)
        t_gen = time.perf_counter() - t0
        t0 = time.perf_counter()
        S, sc = rs.column_scale(Ar)
        t_scale = time.perf_counter() - t0
        t0 = time.perf_counter()
        f = rs.ilup_factorize(S, rs.IlupParams(p=10, tau=0.0, mu=1.0))
        t_ilup = time.perf_counter() - t0
        ent = factor_digests(S.values, sc.scale, f)
        ent.update({"generator": "paper_2603_28642_b200.workloads.config4(seed=4, n=n, nrhs=0)",
                    "params": {"p": 10, "tau": 0.0, "mu": 1.0, "small": 1e-10},
                    "reference_seconds": {"generate": t_gen, "column_scale": t_scale, "ilup": t_ilup},
                    "numpy": np.__version__})
        table[str(n)] = ent
        with open(OUT, "w") as fh:
            json.dump(table, fh, indent=1, sort_keys=True)
        print(f"n={n}: ilup {t_ilup:.1f} s, nnz L1/L2/U {f.L1.nnz}/{f.L2.nnz}/{f.U.nnz}", flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [100000])
