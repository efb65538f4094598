"""Native host setup (csrc/host_setup.cpp) is bit-identical to the reference:
ilup_factorize, build_y_explicit, dense_cholesky_factorize, column_scale."""

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from conftest import csc_from, factors_from, golden, golden_json, reference


def same_csc(a, b):
    return (a.nrows, a.ncols) == (b.nrows, b.ncols) and np.array_equal(a.col_ptr, b.col_ptr) \
        and np.array_equal(a.row_idx, b.row_idx) and np.array_equal(a.values, b.values)


@pytest.mark.parametrize("name", ["cfg0s_mu0.1", "cfg0s_mu1.0", "cfg1s_mu1.0"])
def test_native_setup_matches_reference_fixtures(name):
    from paper_2603_28642_b200 import workloads as W

    z = golden(f"{name}.npz")
    meta = golden_json(f"{name}_reports.json")
    A, b = W.config0(seed=0, m=600, n=400) if name.startswith("cfg0") else W.config1(seed=1, g=24)
    assert np.array_equal(b, z["b"])
    S, sc = P.column_scale(A)
    assert same_csc(S, csc_from(z, "S")) and np.array_equal(sc.scale, z["scale"])
    f = P.ilup_factorize(S, P.IlupParams(**meta["params"]))
    want = factors_from(z)
    assert np.array_equal(f.row_perm.perm, want.row_perm.perm)
    assert same_csc(f.L1, want.L1) and same_csc(f.L2, want.L2) and same_csc(f.U, want.U)
    assert f.nmod == want.nmod and np.array_equal(f.row_counts_final, want.row_counts_final)
    for mode in meta["reports"]:
        if f"Y_{mode}_shape" in z:
            assert same_csc(P.build_y_explicit(f), csc_from(z, f"Y_{mode}"))
        if f"G_{mode}" in z:
            pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
            assert np.array_equal(pre.S_factor.a, z[f"G_{mode}"])


def test_native_ilup_random_vs_live_reference():
    rs = reference()
    rng = np.random.default_rng(31)
    for t in range(40):
        m = int(rng.integers(2, 70))
        n = int(rng.integers(1, m + 1))
        a = rng.standard_normal((m, n)) * (rng.random((m, n)) < rng.uniform(0.05, 1.0))
        if t % 5 == 0 and n > 2:
            a[:, 1] = a[:, 0]  # rank deficient: modified pivots
        for j in range(n):
            if not a[:, j].any():
                a[rng.integers(0, m), j] = 1.0
        prm = dict(p=int(rng.integers(1, 12)), tau=float(rng.choice([0.0, 1e-2, 0.3])),
                   mu=float(rng.choice([0.1, 0.5, 1.0])))
        fr = rs.ilup_factorize(rs.CscMatrix.from_dense(a), rs.IlupParams(**prm))
        fp = P.ilup_factorize(P.CscMatrix.from_dense(a), P.IlupParams(**prm))
        assert np.array_equal(fr.row_perm.perm, fp.row_perm.perm)
        for k in ("L1", "L2", "U"):
            assert same_csc(getattr(fr, k), getattr(fp, k)), (t, k)
        assert fr.nmod == fp.nmod
        assert same_csc(rs.build_y_explicit(fr), P.build_y_explicit(fp))


def test_ilup_validation():
    with pytest.raises(ValueError):
        P.IlupParams(p=0)
    with pytest.raises(ValueError):
        P.IlupParams(mu=0.0)
    with pytest.raises(ValueError):
        P.ilup_factorize(P.CscMatrix.from_dense(np.ones((2, 3))))
    with pytest.raises(np.linalg.LinAlgError):
        P.dense_cholesky_factorize(P.DenseMatrix(np.array([[1.0, 2.0], [2.0, 1.0]])))
    with pytest.raises(ValueError):
        P.column_scale(P.CscMatrix.from_coo(3, 2, [0], [0], [1.0]))


def test_cholesky_hand_cases():
    assert np.array_equal(P.dense_cholesky_factorize(P.DenseMatrix(np.eye(3))).a, np.eye(3))
    f = P.dense_cholesky_factorize(P.DenseMatrix(np.array([[4.0, 2.0], [2.0, 5.0]])))
    assert np.allclose(f.a, [[2.0, 0.0], [1.0, 2.0]], rtol=0, atol=1e-15)
