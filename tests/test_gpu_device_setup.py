"""Device-side setup (csrc/devsetup.cu): large matrices are checked and
converted -- the CSR included -- on the device, and wide triangular
schedules (order > 2^20) are analysed there.  Schedules and results must be
the host path's, bit for bit (analysis.cpp; RSB_HOST_ANALYSIS /
RSB_DEVICE_UPLOAD=0 force it), and the reference's error behaviour kept.
"""

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from oracle import oracle as O
from paper_2603_28642_b200 import _lib as L
from paper_2603_28642_b200.device import DeviceMatrix, get_context

pytestmark = pytest.mark.gpu

N_BIG = (1 << 20) + 4321  # past the single-CTA limit: device analysis


def banded_lower(n, k, rng, diag=True):
    """n x n lower triangular with k random sub-diagonal entries per column
    within a window (wide, shallow level sets) and an optional diagonal."""
    cols = np.repeat(np.arange(n, dtype=np.int64), k)
    rows = cols + rng.integers(1, 5000, size=n * k)
    keep = rows < n
    rows, cols = rows[keep], cols[keep]
    vals = rng.standard_normal(len(rows)) * 0.3
    if diag:
        rows = np.concatenate([rows, np.arange(n)])
        cols = np.concatenate([cols, np.arange(n)])
        vals = np.concatenate([vals, rng.uniform(1.0, 2.0, n) * rng.choice([-1.0, 1.0], n)])
    return P.CscMatrix.from_coo(n, n, rows, cols, vals)


def transpose(M):
    cols = np.repeat(np.arange(M.ncols, dtype=np.int64), np.diff(M.col_ptr))
    return P.CscMatrix.from_coo(M.ncols, M.nrows, cols, M.row_idx, M.values)


def solve(M, kind, b, env, monkeypatch):
    with monkeypatch.context() as m:
        for k, v in env.items():
            m.setenv(k, v)
        dm = DeviceMatrix(P.CscMatrix(M.nrows, M.ncols, M.col_ptr, M.row_idx, M.values), get_context())
        x = np.empty(M.ncols)
        L.check(L.lib().rsb_trsv(dm.h, kind, L.ptr(np.ascontiguousarray(b)), L.ptr(x), L.RSB_HOST))
        lv = dm.levels(kind)
    return x, lv


@pytest.fixture(scope="module")
def mats():
    rng = np.random.default_rng(11)
    Ls = banded_lower(N_BIG, 3, rng, diag=False)  # strictly lower (unit kinds)
    Ln = banded_lower(N_BIG, 3, rng, diag=True)
    return Ls, Ln, transpose(Ln), rng.standard_normal(N_BIG)


@pytest.mark.parametrize("kind", range(6))
def test_device_analysis_matches_host_analysis(mats, kind, monkeypatch):
    Ls, Ln, U, b = mats
    M = {L.TRI_LOWER_UNIT: Ls, L.TRI_LOWER_T_UNIT: Ls, L.TRI_LOWER: Ln, L.TRI_LOWER_T: Ln,
         L.TRI_UPPER: U, L.TRI_UPPER_T: U}[kind]
    xd, lvd = solve(M, kind, b, {}, monkeypatch)
    xh, lvh = solve(M, kind, b, {"RSB_HOST_ANALYSIS": "1", "RSB_DEVICE_UPLOAD": "0"}, monkeypatch)
    assert lvd == lvh, "level count / widest level differ"
    assert np.array_equal(xd, xh), "device-analysed solve differs from the host-analysed one"
    if kind == L.TRI_LOWER:
        assert np.array_equal(xd, O.sparse_lower_solve(Ln, b))


def test_device_upload_products_bitwise():
    """A matrix of >= 2^22 entries (device CSC checks + CSR build): both
    products equal the oracle's bit for bit."""
    rng = np.random.default_rng(5)
    m, n, k = 900_000, 600_000, 7
    rows = rng.integers(0, m, size=n * k)
    cols = np.repeat(np.arange(n, dtype=np.int64), k)
    A = P.CscMatrix.from_coo(m, n, rows, cols, rng.standard_normal(n * k))
    assert A.nnz >= 1 << 22
    x, y = rng.standard_normal(n), rng.standard_normal(m)
    assert np.array_equal(P.matvec(A, x), O.matvec(A, x))
    assert np.array_equal(P.matvec_transpose(A, y), O.matvec_transpose(A, y))


def test_device_upload_rejects_bad_input():
    rng = np.random.default_rng(6)
    n, k = 700_000, 7
    cp = np.arange(0, n * k + 1, k, dtype=np.int64)
    ri = rng.integers(0, n, size=n * k).astype(np.int64)
    ri[123456] = n + 5  # out of range
    with pytest.raises(ValueError, match="row index out of range"):
        DeviceMatrix(P.CscMatrix(n, n, cp, ri, np.ones(n * k)), get_context())
    ri[123456] = 3
    cp2 = cp.copy()
    cp2[1000] = cp2[1001] + 1  # decreasing
    with pytest.raises(ValueError, match="non-decreasing"):
        DeviceMatrix(P.CscMatrix(n, n, cp2, ri, np.ones(n * k)), get_context())


def test_device_analysis_zero_diagonal(mats):
    """A zero diagonal past the single-CTA limit raises LinAlgError, naming
    the first column the reference visits (sc.py:257,274)."""
    _, Ln, _, b = mats
    v = Ln.values.copy()
    first = np.asarray(Ln.col_ptr[:-1])  # lower: the diagonal is stored first in each column
    v[first[777]] = 0.0
    v[first[555]] = 0.0
    Z = P.CscMatrix(Ln.nrows, Ln.ncols, Ln.col_ptr, Ln.row_idx, v)
    with pytest.raises(np.linalg.LinAlgError, match="column 555"):
        P.sparse_lower_solve(Z, b)


def test_banded_transposed_product_bitwise(monkeypatch):
    """A^T y with the gathered vector past 40 MB and RSB_BANDS=1 runs the row-banded product
    (products band by band, then each column's pairwise sum in its original
    order): equal to the oracle, including columns longer than 128 entries
    (numpy's pairwise split) that straddle bands, and in the plain-kernel
    order on another stream (the scratch belongs to the matrix's own)."""
    monkeypatch.setenv("RSB_BANDS", "1")  # opt-in (measured slower at config 4)
    rng = np.random.default_rng(9)
    m, n, k = 6_000_000, 900_000, 5
    rows = rng.integers(0, m, size=n * k)
    cols = np.repeat(np.arange(n, dtype=np.int64), k)
    # a few long columns spanning every band
    long_cols = np.repeat(np.arange(10, dtype=np.int64), 300)
    rows = np.concatenate([rows, rng.integers(0, m, size=len(long_cols))])
    cols = np.concatenate([cols, long_cols])
    A = P.CscMatrix.from_coo(m, n, rows, cols, rng.standard_normal(len(rows)))
    y = rng.standard_normal(m)
    want = O.matvec_transpose(A, y)
    assert np.array_equal(P.matvec_transpose(A, y), want)
    from paper_2603_28642_b200.device import Context

    other = Context()
    dA = DeviceMatrix(A, get_context())
    z = np.empty(n)
    L.check(L.lib().rsb_matvec_transpose(dA.h, L.ptr(y), L.ptr(z), L.RSB_HOST))
    assert np.array_equal(z, want)
    assert other.h is not None
