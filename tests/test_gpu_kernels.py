"""Parity of the sm_100a kernels with the oracle (bit-exact), through the C ABI.

Each test compares the device result of one kernel with the oracle's
restatement of the reference on the same seeded inputs: the golden fixtures
produced by the reference itself, random cases, and the reference's own
edge cases (identity, Lauchli, empty columns, missing diagonals, shape
errors -- pkg/tests/test_sparse_core.py:74-239).
"""

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from conftest import csc_from, golden
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def csc(a):
    return P.CscMatrix.from_dense(np.asarray(a, dtype=float))


@pytest.fixture(scope="module")
def K():
    return golden("kernels.npz")


def test_spmv_golden_bitwise(K):
    c = 0
    while f"mv{c}_shape" in K:
        A = csc_from(K, f"mv{c}")
        assert np.array_equal(P.matvec(A, K[f"mv{c}_x"]), K[f"mv{c}_Ax"]), c
        assert np.array_equal(P.matvec_transpose(A, K[f"mv{c}_y"]), K[f"mv{c}_ATy"]), c
        c += 1


def test_triangular_golden_bitwise(K):
    c = 0
    while f"tl{c}_shape" in K:
        Ls, Ln, U = csc_from(K, f"tl{c}"), csc_from(K, f"tn{c}"), csc_from(K, f"tu{c}")
        b = K[f"t{c}_b"]
        assert np.array_equal(P.sparse_lower_solve(Ls, b, unit_diag=True), K[f"t{c}_lower_unit"]), c
        assert np.array_equal(P.sparse_lower_solve(Ln, b), K[f"t{c}_lower"]), c
        assert np.array_equal(P.sparse_upper_solve(U, b), K[f"t{c}_upper"]), c
        assert np.array_equal(P.sparse_lower_solve_transpose(Ls, b, unit_diag=True), K[f"t{c}_lower_t_unit"]), c
        assert np.array_equal(P.sparse_lower_solve_transpose(Ln, b), K[f"t{c}_lower_t"]), c
        assert np.array_equal(P.sparse_upper_solve_transpose(U, b), K[f"t{c}_upper_t"]), c
        c += 1


def test_cholesky_solve_golden_bitwise(K):
    c = 0
    while f"ch{c}_S" in K:
        assert np.array_equal(P.dense_cholesky_factorize(P.DenseMatrix(K[f"ch{c}_S"])).a, K[f"ch{c}_G"])
        assert np.array_equal(P.dense_cholesky_solve(K[f"ch{c}_G"], K[f"ch{c}_b"]), K[f"ch{c}_x"]), c
        c += 1


@pytest.mark.parametrize("seed", range(6))
def test_kernels_random_vs_oracle(seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(8):
        m, n = int(rng.integers(1, 400)), int(rng.integers(1, 300))
        a = rng.standard_normal((m, n)) * (rng.random((m, n)) < rng.uniform(0.005, 0.9))
        A = csc(a)
        x, y = rng.standard_normal(n), rng.standard_normal(m)
        assert np.array_equal(P.matvec(A, x), O.matvec(A, x))
        assert np.array_equal(P.matvec_transpose(A, y), O.matvec_transpose(A, y))
        k = min(m, n)
        low = np.tril(a[:k, :k], -1) * (rng.random((k, k)) < 0.5)
        up = np.triu(a[:k, :k], 1) + np.diag(rng.uniform(1, 2, k))
        b = rng.standard_normal(k)
        Ls, Ln, U = csc(low), csc(low + np.diag(rng.uniform(1, 2, k))), csc(up)
        assert np.array_equal(P.sparse_lower_solve(Ls, b, True), O.sparse_lower_solve(Ls, b, True))
        assert np.array_equal(P.sparse_lower_solve(Ln, b), O.sparse_lower_solve(Ln, b))
        assert np.array_equal(P.sparse_upper_solve(U, b), O.sparse_upper_solve(U, b))
        assert np.array_equal(P.sparse_lower_solve_transpose(Ls, b, True), O.sparse_lower_solve_transpose(Ls, b, True))
        assert np.array_equal(P.sparse_lower_solve_transpose(Ln, b), O.sparse_lower_solve_transpose(Ln, b))
        assert np.array_equal(P.sparse_upper_solve_transpose(U, b), O.sparse_upper_solve_transpose(U, b))


def test_long_rows_and_columns():
    """Columns longer than numpy's 128 pairwise block, dense rows, L^T columns
    of >= 16 entries (the BLAS-blocked dot inside the transpose solve)."""
    rng = np.random.default_rng(7)
    a = rng.standard_normal((700, 300)) * (rng.random((700, 300)) < 0.8)
    A = csc(a)
    x, y = rng.standard_normal(300), rng.standard_normal(700)
    assert np.array_equal(P.matvec(A, x), O.matvec(A, x))
    assert np.array_equal(P.matvec_transpose(A, y), O.matvec_transpose(A, y))
    low = np.tril(rng.standard_normal((120, 120)), -1) * 0.05
    L = csc(low)
    b = rng.standard_normal(120)
    assert np.array_equal(P.sparse_lower_solve_transpose(L, b, True), O.sparse_lower_solve_transpose(L, b, True))
    up = np.triu(rng.standard_normal((120, 120)), 1) * 0.05 + np.eye(120) * 2
    U = csc(up)
    assert np.array_equal(P.sparse_upper_solve_transpose(U, b), O.sparse_upper_solve_transpose(U, b))
    assert np.array_equal(P.sparse_upper_solve(U, b), O.sparse_upper_solve(U, b))


def test_deep_chain_dag():
    """A bidiagonal L: n dependency levels, one task per level (worst case for
    the sync-free solve), plus the widest DAG (diagonal only)."""
    n = 5000
    rows = np.arange(1, n)
    Lc = P.CscMatrix.from_coo(n, n, rows, rows - 1, np.full(n - 1, -0.5))
    b = np.random.default_rng(3).standard_normal(n)
    got = P.sparse_lower_solve(Lc, b, unit_diag=True)
    assert np.array_equal(got, O.sparse_lower_solve(Lc, b, True))
    assert P.triangular_levels(Lc, 1) == (n, 1)
    assert np.array_equal(P.sparse_lower_solve_transpose(Lc, b, True), O.sparse_lower_solve_transpose(Lc, b, True))
    D = P.CscMatrix.identity(n)
    assert np.array_equal(P.sparse_upper_solve(D, b), b)
    assert P.triangular_levels(D, 2)[0] == 1


def test_reference_hand_cases():
    """pkg/tests/test_sparse_core.py:74-178 on the device."""
    A = P.CscMatrix.identity(2)
    assert np.array_equal(P.matvec(A, [3.0, -1.0]), [3.0, -1.0])
    assert np.array_equal(P.matvec_transpose(A, [3.0, -1.0]), [3.0, -1.0])
    la = csc([[1.0, 1.0], [1e-4, 0.0], [0.0, 1e-4]])
    assert np.array_equal(P.matvec(la, [1.0, 1.0]), [2.0, 1e-4, 1e-4])
    a = np.zeros((3, 3))
    a[0, 0] = 2.0
    assert np.array_equal(P.matvec_transpose(csc(a), [1.0, 1.0, 1.0]), [2.0, 0.0, 0.0])
    Lh = P.CscMatrix(2, 2, [0, 1, 1], [1], [2.0])
    assert np.array_equal(P.sparse_lower_solve(Lh, [1.0, 4.0], unit_diag=True), [1.0, 2.0])
    assert np.array_equal(P.sparse_upper_solve(csc([[2.0, 1.0], [0.0, 3.0]]), [5.0, 6.0]), [1.5, 2.0])
    assert np.array_equal(P.sparse_lower_solve(csc([[1.0, 0.0], [5.0, 1.0]]), [1.0, 6.0]), [1.0, 1.0])


def test_errors_match_reference():
    A = P.CscMatrix.identity(3)
    with pytest.raises(ValueError):
        P.matvec(A, [1.0, 2.0])
    with pytest.raises(ValueError):
        P.matvec_transpose(A, [1.0, 2.0])
    with pytest.raises(np.linalg.LinAlgError):
        P.sparse_upper_solve(P.CscMatrix(2, 2, [0, 1, 1], [0], [1.0]), [1.0, 1.0])
    with pytest.raises(np.linalg.LinAlgError):
        P.sparse_lower_solve(P.CscMatrix(2, 2, [0, 1, 2], [1, 1], [5.0, 1.0]), [1.0, 1.0])
    with pytest.raises(ValueError):
        P.sparse_lower_solve(P.CscMatrix.from_coo(2, 3, [], [], []), [1.0, 1.0])
    with pytest.raises(ValueError):
        P.sparse_upper_solve(A, [1.0])


def test_nan_and_signed_zero_propagation():
    """Skip-on-zero and -0.0 handling follow the reference exactly."""
    L = P.CscMatrix(3, 3, [0, 2, 3, 3], [1, 2, 2], [-1.0, 2.0, 3.0])
    for b in ([0.0, -0.0, 1.0], [-0.0, 0.0, -0.0], [np.inf, 1.0, 0.0], [np.nan, 0.0, 1.0], [0.0, np.inf, 1.0]):
        b = np.array(b)
        got = P.sparse_lower_solve(L, b, True)
        want = O.sparse_lower_solve(L, b, True)
        assert np.array_equal(got.view(np.int64), want.view(np.int64)) or np.array_equal(got, want, equal_nan=True)


def test_power_method_matches_oracle():
    rng = np.random.default_rng(11)
    a = rng.standard_normal((300, 120)) * (rng.random((300, 120)) < 0.1)
    for j in range(120):
        if not a[:, j].any():
            a[0, j] = 1.0
    A = csc(a)
    assert P.power_method_norm2(A, 100, 3) == O.power_method_norm2(A, 100, 3)
    assert P.power_method_norm2(P.CscMatrix.from_coo(4, 3, [], [], []), 5, 0) == 0.0
    with pytest.raises(ValueError):
        P.power_method_norm2(A, 0)


@pytest.mark.parametrize("n", [1, 15, 16, 17, 31, 32, 33, 48, 100, 1000, 12287, 12288, 12303, 12320, 32 * 256 + 31,
                               32 * (1024 * 3 + 16 * 5 + 7) + 20, 65536, 98304, 1_000_003, 1_500_000])
def test_device_dot_reference_order(n):
    from paper_2603_28642_b200 import _lib as L
    from paper_2603_28642_b200.device import get_context

    rng = np.random.default_rng(n)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    out = np.zeros(1)
    L.check(L.lib().rsb_dot(get_context().h, n, L.ptr(a), L.ptr(b), out.ctypes.data_as(L.f64p), L.RSB_HOST))
    assert out[0] == O.dot(a, b)


_SPMV_VARIANT_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {repo!r}); sys.path.insert(0, {tests!r})
import paper_2603_28642_b200 as P
from paper_2603_28642_b200 import workloads as W
from conftest import csc_from, golden
from oracle import oracle as O
K = golden("kernels.npz")
mats = []
c = 0
while f"mv{{c}}_shape" in K:
    mats.append(csc_from(K, f"mv{{c}}")); c += 1
mats.append(W.config4(seed=4, n=5000, nrhs=0)[0])
mats.append(W.config2(seed=2, n=3000)[0])
rng = np.random.default_rng(7)
for A in mats:
    x, y = rng.standard_normal(A.ncols), rng.standard_normal(A.nrows)
    assert np.array_equal(P.matvec(A, x), O.matvec(A, x))
    assert np.array_equal(P.matvec_transpose(A, y), O.matvec_transpose(A, y))
print("ok")
"""


@pytest.mark.parametrize("variant", ["tile", "thread"])
def test_spmv_forced_variants_bitwise(variant):
    """Both SpMV kernel families (tiled / thread per line, RSB_SPMV) on the
    golden matrices, config 4 (6 entries per row) and config 2 (dense rows
    past the tile's staging buffer)."""
    import os
    import subprocess
    import sys

    tests = os.path.dirname(os.path.abspath(__file__))
    script = _SPMV_VARIANT_SCRIPT.format(repo=os.path.dirname(tests), tests=tests)
    r = subprocess.run([sys.executable, "-c", script], env=dict(os.environ, RSB_SPMV=variant),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
