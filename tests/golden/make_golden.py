"""Generate the golden fixtures in tests/golden/ by running the REFERENCE
package (`rowsplit`, read-only at /root/reference/pkg/src) in this container.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden.py

The reference cannot travel to the GPU box, so its outputs on seeded inputs
are committed here; tests/test_oracle_pin.py and tests/test_host_setup.py
pin the oracle and the native host setup against them.  Inputs are
regenerated from seeds wherever possible so the fixtures stay small.
"""

from __future__ import annotations

import json
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

import numpy as np  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import rowsplit as rs  # noqa: E402

from paper_2603_28642_b200 import workloads as W  # noqa: E402


def csc_arrays(prefix, M):
    return {f"{prefix}_shape": np.array([M.nrows, M.ncols]), f"{prefix}_ptr": M.col_ptr,
            f"{prefix}_idx": M.row_idx, f"{prefix}_val": M.values}


def random_csc(rng, m, n, dens):
    a = rng.standard_normal((m, n)) * (rng.random((m, n)) < dens)
    return rs.CscMatrix.from_dense(a)


def kernels_fixture():
    """matvec / matvec_transpose / the four triangular solves / dense Cholesky
    on seeded random inputs, including long columns (> 128 entries, numpy's
    pairwise split) and BLAS dots of length >= 16."""
    rng = np.random.default_rng(20261020)
    out = {}
    cases = [(7, 5, 0.4), (50, 40, 0.3), (300, 200, 0.05), (400, 3, 0.9), (3, 300, 0.9), (1, 1, 1.0),
             (260, 150, 0.6)]
    for c, (m, n, dens) in enumerate(cases):
        A = random_csc(rng, m, n, dens)
        x = rng.standard_normal(n)
        y = rng.standard_normal(m)
        out.update(csc_arrays(f"mv{c}", A))
        out[f"mv{c}_x"], out[f"mv{c}_y"] = x, y
        out[f"mv{c}_Ax"] = rs.matvec(A, x)
        out[f"mv{c}_ATy"] = rs.matvec_transpose(A, y)
    tri = [(6, 0.6), (40, 0.3), (120, 0.5), (200, 0.1)]
    for c, (k, dens) in enumerate(tri):
        low = np.tril(rng.standard_normal((k, k)), -1) * (rng.random((k, k)) < dens)
        up = np.triu(rng.standard_normal((k, k)), 1) * (rng.random((k, k)) < dens) + np.diag(
            rng.uniform(1, 2, k) * rng.choice([-1.0, 1.0], k))
        Ls = rs.CscMatrix.from_dense(low)
        Ln = rs.CscMatrix.from_dense(low + np.diag(rng.uniform(1, 2, k)))
        U = rs.CscMatrix.from_dense(up)
        b = rng.standard_normal(k)
        out.update(csc_arrays(f"tl{c}", Ls))
        out.update(csc_arrays(f"tn{c}", Ln))
        out.update(csc_arrays(f"tu{c}", U))
        out[f"t{c}_b"] = b
        out[f"t{c}_lower_unit"] = rs.sparse_lower_solve(Ls, b, unit_diag=True)
        out[f"t{c}_lower"] = rs.sparse_lower_solve(Ln, b)
        out[f"t{c}_upper"] = rs.sparse_upper_solve(U, b)
        out[f"t{c}_lower_t_unit"] = rs.sparse_lower_solve_transpose(Ls, b, unit_diag=True)
        out[f"t{c}_lower_t"] = rs.sparse_lower_solve_transpose(Ln, b)
        out[f"t{c}_upper_t"] = rs.sparse_upper_solve_transpose(U, b)
    for c, s in enumerate([1, 5, 40, 150]):
        yv = rng.standard_normal((s, s + 3))
        S = np.eye(s) + yv @ yv.T
        f = rs.dense_cholesky_factorize(rs.DenseMatrix(S))
        b = rng.standard_normal(s)
        out[f"ch{c}_S"] = S
        out[f"ch{c}_G"] = f.a
        out[f"ch{c}_b"] = b
        out[f"ch{c}_x"] = rs.dense_cholesky_solve(f, b)
    # BLAS dot association: vectors regenerated from the seed in the test
    lens = list(range(1, 80)) + [100, 127, 128, 129, 255, 256, 1000, 4097, 9999]
    drng = np.random.default_rng(77)
    dots = []
    for n in lens:
        a, b = drng.standard_normal(n), drng.standard_normal(n)
        dots.append(a @ b)
    out["dot_lens"] = np.array(lens)
    out["dot_vals"] = np.array(dots)
    # numpy pairwise summation via reduceat on long segments
    seg = drng.standard_normal(5000)
    starts = np.array([0, 3, 11, 150, 400, 1700, 1701])
    out["pw_seg"] = seg
    out["pw_starts"] = starts
    out["pw_sums"] = np.add.reduceat(seg, starts)
    return out


def solve_fixture(name, A, b, params, modes, delta, max_iters, rs_seed=0):
    """Scaled matrix + reference factors + Y + S factor + apply outputs +
    pcgls outputs for each coupling mode."""
    out = {}
    Ar = rs.CscMatrix(A.nrows, A.ncols, A.col_ptr, A.row_idx, A.values)
    S, scaling = rs.column_scale(Ar)
    norm_a = rs.power_method_norm2(S, 100, rs_seed)
    out.update(csc_arrays("S", S))
    out["scale"] = scaling.scale
    out["b"] = b
    out["norm_a"] = np.array(norm_a)
    f = rs.ilup_factorize(S, rs.IlupParams(**params))
    out["perm"] = f.row_perm.perm
    out.update(csc_arrays("L1", f.L1))
    out.update(csc_arrays("L2", f.L2))
    out.update(csc_arrays("U", f.U))
    out["nmod"] = np.array(f.nmod)
    out["row_counts"] = f.row_counts_final
    rng = np.random.default_rng(99)
    n, s = S.ncols, S.nrows - S.ncols
    r1, r2 = rng.standard_normal(n), rng.standard_normal(s)
    out["r1"], out["r2"] = r1, r2
    reports = {}
    for mode in modes:
        pre = rs.build_preconditioner(f, s_mode=rs.SMode(mode))
        if pre.Y is not None:
            out.update(csc_arrays(f"Y_{mode}", pre.Y))
        if pre.S_factor is not None:
            out[f"G_{mode}"] = pre.S_factor.a
        out[f"h_{mode}"] = pre.apply(r1, r2)
        out[f"yapply_{mode}"] = pre.y_apply(r1)
        out[f"yapplyT_{mode}"] = pre.y_apply_transpose(r2)
        out[f"smv_{mode}"] = pre.s_matvec_implicit(r2)
        x, rep = rs.pcgls(S, b, pre, rs.CglsConfig(norm_A=norm_a, delta=delta, max_iters=max_iters))
        out[f"x_{mode}"] = x
        reports[mode] = rep.to_dict()
    x, rep = rs.pcgls(S, b, None, rs.CglsConfig(norm_A=norm_a, delta=delta, max_iters=max_iters))
    out["x_plain"] = x
    reports["plain"] = rep.to_dict()
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    with open(os.path.join(HERE, f"{name}_reports.json"), "w") as fh:
        json.dump({"params": params, "delta": delta, "max_iters": max_iters, "reports": reports}, fh,
                  indent=1, sort_keys=True)


def identity_fixture():
    """The reference's 5x5-identity golden case (pkg/tests/test_cli.py:54-58,
    pkg/tests/data/golden_identity.json): dense mode, delta 1e-10; pins the
    stopped-early partial-window branch (history [1.0, 0.0])."""
    A = rs.CscMatrix.identity(5)
    b = np.random.default_rng(42).uniform(-1.0, 1.0, 5)
    S, _ = rs.column_scale(A)
    norm_a = rs.power_method_norm2(S, 100, 42)
    f = rs.ilup_factorize(S, rs.IlupParams())
    pre = rs.build_preconditioner(f, s_mode=rs.SMode.DENSE_FACTOR)
    x, rep = rs.pcgls(S, b, pre, rs.CglsConfig(norm_A=norm_a, delta=1e-10))
    with open(os.path.join(HERE, "identity5.json"), "w") as fh:
        json.dump({"b": b.tolist(), "norm_a": norm_a, "x": x.tolist(), "report": rep.to_dict()}, fh,
                  indent=1, sort_keys=True)


def main():
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kernels_fixture())
    A, b = W.config0(seed=0, m=600, n=400)
    for mu in (0.1, 1.0):
        solve_fixture(f"cfg0s_mu{mu}", A, b, dict(p=10, tau=1e-3, mu=mu), ["dense", "cg", "identity"],
                      1e-8, 60)
    A, b = W.config1(seed=1, g=24)
    solve_fixture("cfg1s_mu1.0", A, b, dict(p=10, tau=0.0, mu=1.0), ["cg", "identity"], 1e-10, 80)
    identity_fixture()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
