"""Parity of the device preconditioner application with the oracle / reference.

The golden fixtures hold the reference's own apply, y_apply,
y_apply_transpose and s_matvec_implicit outputs on seeded configs (default
mu = 0.1 and mu = 1.0 factors); the device must reproduce them bit for bit.
The reference's behavioural tests (pkg/tests/test_precond.py:192-266) run
on the device too.
"""

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from conftest import csc_from, factors_from, golden, golden_json, rel_err
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def csc(a):
    return P.CscMatrix.from_dense(np.asarray(a, dtype=float))


@pytest.mark.parametrize("name", ["cfg0s_mu0.1", "cfg0s_mu1.0", "cfg1s_mu1.0"])
def test_apply_golden_bitwise(name):
    z = golden(f"{name}.npz")
    meta = golden_json(f"{name}_reports.json")
    f = factors_from(z)
    for mode in meta["reports"]:
        if mode == "plain":
            continue
        pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
        if f"Y_{mode}_shape" in z:  # native setup reproduces the reference's Y and S factor
            Y = csc_from(z, f"Y_{mode}")
            assert np.array_equal(pre.Y.col_ptr, Y.col_ptr) and np.array_equal(pre.Y.values, Y.values)
        if f"G_{mode}" in z:
            assert np.array_equal(pre.S_factor.a, z[f"G_{mode}"])
        assert np.array_equal(pre.apply(z["r1"], z["r2"]), z[f"h_{mode}"]), mode
        assert np.array_equal(pre.y_apply(z["r1"]), z[f"yapply_{mode}"]), mode
        assert np.array_equal(pre.y_apply_transpose(z["r2"]), z[f"yapplyT_{mode}"]), mode
        assert np.array_equal(pre.s_matvec_implicit(z["r2"]), z[f"smv_{mode}"]), mode


@pytest.mark.parametrize("mu", [0.1, 1.0])
@pytest.mark.parametrize("mode", ["dense", "cg", "identity"])
@pytest.mark.parametrize("ymode", ["explicit", "implicit"])
def test_apply_vs_oracle_config0(mu, mode, ymode):
    from paper_2603_28642_b200 import workloads as W

    if mode == "dense" and ymode == "implicit":
        pytest.skip("dense S requires the explicit Y")
    A, _ = W.config0(seed=5, m=900, n=600)
    S, _ = P.column_scale(A)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=1e-3, mu=mu))
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode), y_mode=P.YMode(ymode), cg_iters=3)
    op = O.OraclePreconditioner.from_reference(pre)
    rng = np.random.default_rng(int(mu * 10))
    r1, r2 = rng.standard_normal(600), rng.standard_normal(300)
    assert np.array_equal(pre.apply(r1, r2), op.apply(r1, r2))
    assert np.array_equal(pre.y_apply(r1), op.y_apply(r1))
    assert np.array_equal(pre.y_apply_transpose(r2), op.y_apply_transpose(r2))
    assert np.array_equal(pre.s_matvec_implicit(r2), op.s_matvec_implicit(r2))


def test_apply_square_degenerates_to_triangular_solves():
    """pkg/tests/test_precond.py:192-199 (atol 0)."""
    rng = np.random.default_rng(8)
    f = P.ilup_factorize(csc(rng.standard_normal((6, 6))), P.IlupParams(p=6, mu=0.1))
    pre = P.build_preconditioner(f, s_mode=P.SMode.DENSE_FACTOR)
    r1 = rng.standard_normal(6)
    h = pre.apply(r1, np.zeros(0))
    assert np.array_equal(h, P.sparse_upper_solve(f.U, P.sparse_lower_solve(f.L1, r1, unit_diag=True)))


def test_apply_exact_factors_give_lls_solution():
    """pkg/tests/test_precond.py:202-214."""
    rng = np.random.default_rng(9)
    for _ in range(10):
        n = int(rng.integers(3, 10))
        m = n + int(rng.integers(0, 3))
        a = rng.standard_normal((m, n))
        f = P.ilup_factorize(csc(a), P.IlupParams(p=m, mu=0.1))
        pre = P.build_preconditioner(f, s_mode=P.SMode.DENSE_FACTOR)
        b = rng.uniform(-1, 1, m)
        pb = b[f.row_perm.perm]
        h = pre.apply(pb[:n], pb[n:])
        want = np.linalg.lstsq(a, b, rcond=None)[0]
        assert rel_err(h, want) <= 1e-10


def test_inner_cg_limit_matches_dense_factor():
    """pkg/tests/test_precond.py:257-266: cg(s) = dense within 1e-8."""
    rng = np.random.default_rng(12)
    for _ in range(6):
        n, s = int(rng.integers(4, 20)), int(rng.integers(1, 16))
        top = np.eye(n) + 0.3 * rng.standard_normal((n, n)) / np.sqrt(n)
        bottom = 0.5 * rng.standard_normal((s, n)) / np.sqrt(n)
        f = P.ilup_factorize(csc(np.vstack([top, bottom])), P.IlupParams(p=n + s, mu=0.1))
        pe = P.build_preconditioner(f, s_mode=P.SMode.DENSE_FACTOR)
        pi = P.build_preconditioner(f, s_mode=P.SMode.INNER_CG, cg_iters=s)
        r1, r2 = rng.standard_normal(n), rng.standard_normal(s)
        assert rel_err(pi.apply(r1, r2), pe.apply(r1, r2)) <= 1e-8


def test_apply_dimension_mismatch_and_modes():
    rng = np.random.default_rng(11)
    f = P.ilup_factorize(csc(rng.standard_normal((7, 4))), P.IlupParams())
    pre = P.build_preconditioner(f, s_mode=P.SMode.IDENTITY)
    with pytest.raises(ValueError):
        pre.apply(np.zeros(4), np.zeros(1))
    with pytest.raises(ValueError):
        P.build_preconditioner(f, s_mode=P.SMode.DENSE_FACTOR, dense_cap=2)
    with pytest.raises(ValueError):
        P.build_preconditioner(f, s_mode=P.SMode.DENSE_FACTOR, y_mode=P.YMode.IMPLICIT)
    with pytest.raises(ValueError):
        P.build_preconditioner(f, cg_iters=0)


def test_s_matvec_zero_l2_and_hand_case():
    """pkg/tests/test_precond.py:108-124."""
    f = P.IlupFactors(P.Permutation.identity(5), P.CscMatrix.from_coo(3, 3, [], [], []),
                      P.CscMatrix.from_coo(2, 3, [], [], []), P.CscMatrix.identity(3), 0,
                      np.zeros(5, dtype=np.int64))
    pre = P.build_preconditioner(f, s_mode=P.SMode.IDENTITY)
    v = np.array([1.5, -2.0])
    assert np.array_equal(pre.s_matvec_implicit(v), v)
    hf = P.IlupFactors(P.Permutation.identity(3), P.CscMatrix.from_coo(2, 2, [], [], []),
                       csc([[1.0, 1.0]]), P.CscMatrix.identity(2), 0, np.zeros(3, dtype=np.int64))
    pre = P.build_preconditioner(hf, s_mode=P.SMode.IDENTITY, y_mode=P.YMode.IMPLICIT)
    assert np.array_equal(pre.s_matvec_implicit([2.0]), [6.0])
    pre = P.build_preconditioner(P.IlupFactors(P.Permutation.identity(3), P.CscMatrix.from_coo(2, 2, [], [], []),
                                               csc([[2.0, 0.0]]), P.CscMatrix.identity(2), 0,
                                               np.zeros(3, dtype=np.int64)), s_mode=P.SMode.DENSE_FACTOR)
    assert np.array_equal(pre.y_apply([3.0, 5.0]), [6.0])


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_inner_cg_step_counts_bitwise(k):
    """_cg_fixed_steps (pc.py:284-310) with k steps: the device skips the last
    step's r / rho_new / p updates (they feed nothing), so w and the apply must
    still equal the oracle bit for bit -- also on applications that follow an
    early break (rho = 0 on a zero u), which must not leak their stop flag."""
    from paper_2603_28642_b200 import workloads as W

    A, _ = W.config0(seed=7, m=600, n=400)
    S, _ = P.column_scale(A)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=1e-3, mu=1.0))
    pre = P.build_preconditioner(f, s_mode=P.SMode.INNER_CG, cg_iters=k)
    op = O.OraclePreconditioner.from_reference(pre)
    rng = np.random.default_rng(k)
    r1, r2 = rng.standard_normal(400), rng.standard_normal(200)
    assert np.array_equal(pre.apply(r1, r2), op.apply(r1, r2))
    assert np.array_equal(pre.s_matvec_implicit(r2), op.s_matvec_implicit(r2))
    # r2 = Y r1 makes u = 0: the inner CG stops at rho == 0 (w = 0)
    u0 = pre.y_apply(r1)
    assert np.array_equal(pre.apply(r1, u0), op.apply(r1, u0))
    # and the next application runs all k steps again
    r1b, r2b = rng.standard_normal(400), rng.standard_normal(200)
    assert np.array_equal(pre.apply(r1b, r2b), op.apply(r1b, r2b))


def test_chol_smem_limit_is_grow_only():
    """Two dense S solves whose vectors need > 48 KB of shared memory: the
    larger one must still launch after the smaller one was prepared
    (kernels.cu prepare_chol keeps the largest granted limit)."""
    for s in (7000, 6200, 7000):
        g = np.eye(s) * 2.0
        b = np.arange(1.0, s + 1.0)
        x = P.dense_cholesky_solve(P.DenseMatrix(g), b)
        assert np.array_equal(x, b / 4.0)
