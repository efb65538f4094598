"""Dense-coupling preconditioner built on the device (csrc/dbuild.cu,
SURVEY.md 8(f)2): explicit Y = L2 L1^{-1} (pc.py:55-82), S = I + Y Y^T
(pc.py:85-92) and its Cholesky factor (sc.py:585-604).

Bars: Y bit-identical to the reference's (fixtures made by the reference,
tests/golden/make_golden.py, and the host build pinned to it); the device
Cholesky bit-identical to the reference's sweep given the same S; S within
1e-13 (max-norm, relative) of numpy's `yd @ yd.T` -- the one step whose
BLAS order is not reproduced; a preconditioner built on the device applies
within 1e-10 of the reference's (the north star's apply tolerance).
"""

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from conftest import factors_from, golden, rel_err
from paper_2603_28642_b200.precond import _gram_plus_identity, dense_build_device

pytestmark = pytest.mark.gpu

S_TOL = 1e-13
APPLY_TOL = 1e-10


def _same_csc(a, b):
    return (a.nrows, a.ncols) == (b.nrows, b.ncols) and np.array_equal(a.col_ptr, b.col_ptr) and \
        np.array_equal(a.row_idx, b.row_idx) and np.array_equal(a.values, b.values)


def _spd(s, seed, cond=1e3):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.standard_normal((s, s)))
    d = np.geomspace(1.0, cond, s)
    a = (q * d) @ q.T
    return np.asfortranarray((a + a.T) / 2)


@pytest.mark.parametrize("name", ["cfg0s_mu0.1.npz", "cfg0s_mu1.0.npz"])
def test_y_s_factor_vs_reference_fixtures(name):
    z = golden(name)
    f = factors_from(z)
    Y, S, F, sec = dense_build_device(f, what=2)
    from conftest import csc_from
    Yref = csc_from(z, "Y_dense")
    assert _same_csc(Y, Yref), "device Y differs from the reference's"
    S_np = _gram_plus_identity(Yref).a
    err = np.max(np.abs(S.a - S_np)) / np.max(np.abs(S_np))
    assert err <= S_TOL, err
    assert np.array_equal(S.a, S.a.T)
    # the factor of the device S equals the host sweep on that S, bit for bit
    assert np.array_equal(F.a, P.dense_cholesky_factorize(S, setup="host").a)
    # and the factor of the reference's own S equals the reference's factor
    # up to the S rounding only
    assert rel_err(F.a, z["G_dense"]) < 1e-10


def test_y_matches_host_build_illc1850():
    z = golden("illc1850.npz")
    f = factors_from(z)
    Y, _, _, _ = dense_build_device(f, what=0)
    assert _same_csc(Y, P.build_y_explicit(f))


@pytest.mark.parametrize("s", [1, 2, 31, 32, 33, 100, 257, 1000])
def test_cholesky_device_bitwise(s):
    a = _spd(s, s)
    assert np.array_equal(P.dense_cholesky_factorize(a, setup="device").a,
                          P.dense_cholesky_factorize(a, setup="host").a)


def test_cholesky_device_not_spd_same_pivot():
    a = _spd(70, 7)
    a[40, 40] = -5.0
    msgs = []
    for where in ("host", "device"):
        with pytest.raises(np.linalg.LinAlgError) as e:
            P.dense_cholesky_factorize(a, setup=where)
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1] and "pivot" in msgs[0]
    b = _spd(5, 1)
    b[2, 2] = np.nan
    with pytest.raises(np.linalg.LinAlgError):
        P.dense_cholesky_factorize(b, setup="device")


def test_cholesky_device_empty():
    assert P.dense_cholesky_factorize(np.zeros((0, 0)), setup="device").a.shape == (0, 0)


@pytest.mark.parametrize("name", ["cfg0s_mu0.1.npz", "cfg0s_mu1.0.npz"])
def test_device_built_preconditioner_applies_like_reference(name):
    z = golden(name)
    f = factors_from(z)
    pre = P.build_preconditioner(f, s_mode=P.SMode.DENSE_FACTOR, setup="device")
    host = P.build_preconditioner(f, s_mode=P.SMode.DENSE_FACTOR, setup="host")
    assert pre.psize == host.psize
    assert _same_csc(pre.Y, host.Y)
    h = pre.apply(z["r1"], z["r2"])
    assert rel_err(h, z["h_dense"]) <= APPLY_TOL
    # explicit Y with the cg coupling needs no S: bitwise to the reference
    pre_cg = P.build_preconditioner(f, s_mode=P.SMode.INNER_CG, y_mode=P.YMode.EXPLICIT, setup="device")
    host_cg = P.build_preconditioner(f, s_mode=P.SMode.INNER_CG, y_mode=P.YMode.EXPLICIT, setup="host")
    assert _same_csc(pre_cg.Y, host_cg.Y) and pre_cg.S_factor is None
    assert np.array_equal(pre_cg.apply(z["r1"], z["r2"]), host_cg.apply(z["r1"], z["r2"]))


def test_device_build_empty_l2_and_bad_setup():
    z = golden("cfg0s_mu1.0.npz")
    f = factors_from(z)
    with pytest.raises(ValueError):
        P.build_preconditioner(f, setup="gpu")
    from paper_2603_28642_b200.types import CscMatrix
    n = f.L1.ncols
    empty = CscMatrix(0, n, np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0))
    f0 = type(f)(f.row_perm, f.L1, empty, f.U, f.nmod, f.row_counts_final)
    Y, S, F, _ = dense_build_device(f0, what=2)
    assert (Y.nrows, Y.ncols, Y.nnz) == (0, n, 0)
    assert S.a.shape == (0, 0) and F.a.shape == (0, 0)


def test_column_scale_device_bitwise():
    """column_scale (sc.py:405-425) on the device against the native host
    version (itself pinned to the reference): short columns, columns longer
    than numpy's pairwise leaf (128) and than its 8-term block, an empty
    column's error."""
    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import workloads as W

    rng = np.random.default_rng(5)
    mats = [W.config4(seed=4, n=20_000, nrhs=0)[0], W.config2(seed=2, n=3000)[0]]
    # one matrix with columns of 1 .. 400 entries
    rows, cols = [], []
    for j, k in enumerate([1, 2, 7, 8, 9, 15, 16, 17, 127, 128, 129, 130, 257, 400]):
        rows += sorted(rng.choice(500, size=k, replace=False).tolist())
        cols += [j] * k
    mats.append(P.CscMatrix.from_coo(500, 14, np.array(rows), np.array(cols), rng.standard_normal(len(rows))))
    for A in mats:
        Sh, ch = P.column_scale(A, setup="host")
        Sd, cd = P.column_scale(A, setup="device")
        assert np.array_equal(Sh.values, Sd.values) and np.array_equal(ch.scale, cd.scale)
        assert np.array_equal(Sh.col_ptr, Sd.col_ptr) and np.array_equal(Sh.row_idx, Sd.row_idx)
    E = P.CscMatrix.from_coo(4, 3, np.array([0, 1]), np.array([0, 2]), np.array([1.0, 2.0]))
    with pytest.raises(ValueError, match="zero column 1"):
        P.column_scale(E, setup="device")
