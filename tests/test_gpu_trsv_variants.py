"""The three triangular-solve kernels against the oracle, bit for bit.

Matrices are built level by level so that each case lands on a chosen
kernel: the lean single-CTA solve (trsv_lean.cu) at every consumer-warp
count and the longest task it takes (16 entries in the sequential order, 15
in the dot order), the staged single-CTA solve past those limits, and the
grid-wide solves for wide DAGs (a launch per level, or sync-free) -- with an odd number of levels, many
chunks, diagonals and right-hand sides outside the exact-division range,
signed zeros, infinities and NaNs.  Every case also runs with the lean
kernel disabled (RSB_TRSV_LEAN=0) and must give the same bits.
"""

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from paper_2603_28642_b200 import _lib as L
from paper_2603_28642_b200.device import DeviceMatrix, get_context
from oracle import oracle as O

pytestmark = pytest.mark.gpu

SOLVES = {
    L.TRI_LOWER_UNIT: (lambda M, b: P.sparse_lower_solve(M, b, unit_diag=True),
                       lambda M, b: O.sparse_lower_solve(M, b, True)),
    L.TRI_LOWER: (lambda M, b: P.sparse_lower_solve(M, b), lambda M, b: O.sparse_lower_solve(M, b, False)),
    L.TRI_UPPER: (P.sparse_upper_solve, O.sparse_upper_solve),
    L.TRI_LOWER_T_UNIT: (lambda M, b: P.sparse_lower_solve_transpose(M, b, unit_diag=True),
                         lambda M, b: O.sparse_lower_solve_transpose(M, b, True)),
    L.TRI_LOWER_T: (lambda M, b: P.sparse_lower_solve_transpose(M, b),
                    lambda M, b: O.sparse_lower_solve_transpose(M, b, False)),
    L.TRI_UPPER_T: (P.sparse_upper_solve_transpose, O.sparse_upper_solve_transpose),
}


def leveled_lower(widths, k, rng, diag=None, window=1500):
    """Lower triangular CSC: unknowns numbered level by level; an unknown of
    level l > 0 depends on one of level l - 1 and up to k - 1 earlier ones
    among the `window` before its level (row lengths 1..k; a window within
    the shared-memory ring keeps the lean kernel eligible); diag(values)
    adds the diagonal."""
    off = np.concatenate([[0], np.cumsum(widths)])
    n = int(off[-1])
    rows, cols, vals = [], [], []
    for l in range(1, len(widths)):
        for t in range(off[l], off[l + 1]):
            deps = {int(rng.integers(off[l - 1], off[l]))}
            want = int(rng.integers(1, k + 1))
            while len(deps) < min(want, t):
                deps.add(int(rng.integers(max(0, off[l] - window), off[l])))
            for d in deps:
                rows.append(t)
                cols.append(d)
                vals.append(rng.standard_normal())
    if diag is not None:
        d = diag(n)
        rows += list(range(n))
        cols += list(range(n))
        vals += list(d)
    return P.CscMatrix.from_coo(n, n, np.array(rows), np.array(cols), np.array(vals))


def transpose(M):
    cols = np.repeat(np.arange(M.ncols), np.diff(M.col_ptr))
    return P.CscMatrix.from_coo(M.ncols, M.nrows, cols, M.row_idx.copy(), M.values.copy())


def same_bits(a, b):
    return np.array_equal(a.view(np.int64), b.view(np.int64)) or np.array_equal(a, b, equal_nan=True)


def variant(M, kind):
    return DeviceMatrix(M, get_context()).variant(kind)


def check(M, kind, b, monkeypatch, expect=None):
    dev, orc = SOLVES[kind]
    want = orc(M, b)
    got = dev(M, b)
    assert same_bits(got, want), kind
    v = variant(M, kind)
    if expect is not None:
        assert v[0] == expect[0] and (expect[1] is None or v[1] == expect[1]), (v, expect)
    with monkeypatch.context() as m:
        m.setenv("RSB_TRSV_LEAN", "0")
        M2 = P.CscMatrix(M.nrows, M.ncols, M.col_ptr.copy(), M.row_idx.copy(), M.values.copy())
        assert variant(M2, kind)[0] != "lean"
        assert same_bits(dev(M2, b), want), kind
    return v


@pytest.mark.parametrize("width", [32, 64, 96, 128])
def test_lean_every_warp_count(width, monkeypatch):
    rng = np.random.default_rng(width)
    M = leveled_lower([width] * 301, 6, rng)  # odd level count
    b = rng.standard_normal(M.ncols)
    check(M, L.TRI_LOWER_UNIT, b, monkeypatch, ("lean", None))


def test_lean_longest_tasks(monkeypatch):
    rng = np.random.default_rng(1)
    M = leveled_lower([32] * 120, 16, rng)
    b = rng.standard_normal(M.ncols)
    assert check(M, L.TRI_LOWER_UNIT, b, monkeypatch)[0] == "lean"  # 16 entries, sequential order
    # dot order: columns of the transposed solve with 15 entries stay lean,
    # 16 or more take another kernel (blocked BLAS order)
    for k, lean in ((15, True), (40, False)):
        rows, cols = [], []
        n = 33 * 40
        for j in range(n - 1):
            for i in sorted(rng.choice(np.arange(j + 1, n), size=min(k, n - j - 1), replace=False)):
                rows.append(i)
                cols.append(j)
        T = P.CscMatrix.from_coo(n, n, np.array(rows), np.array(cols), rng.standard_normal(len(rows)))
        v = check(T, L.TRI_LOWER_T_UNIT, rng.standard_normal(n), monkeypatch)
        assert (v[0] == "lean") == lean, v


def test_wide_levels_use_staged_or_grid(monkeypatch):
    rng = np.random.default_rng(2)
    M = leveled_lower([160] * 40, 5, rng)
    b = rng.standard_normal(M.ncols)
    assert check(M, L.TRI_LOWER_UNIT, b, monkeypatch)[0] in ("staged", "grid", "levels")
    W = leveled_lower([6000] * 5, 4, rng)
    bw = rng.standard_normal(W.ncols)
    assert check(W, L.TRI_LOWER_UNIT, bw, monkeypatch)[0] == "grid"
    # the level-synchronous cooperative kernel on the same DAG
    with monkeypatch.context() as m:
        m.setenv("RSB_TRSV_GRID", "levelsync")
        W0 = P.CscMatrix(W.nrows, W.ncols, W.col_ptr.copy(), W.row_idx.copy(), W.values.copy())
        assert check(W0, L.TRI_LOWER_UNIT, bw, monkeypatch)[0] == "levelsync"
    # the level-synchronous item kernel on the same DAG
    with monkeypatch.context() as m:
        m.setenv("RSB_TRSV_GRID", "lsync")
        W1 = P.CscMatrix(W.nrows, W.ncols, W.col_ptr.copy(), W.row_idx.copy(), W.values.copy())
        assert check(W1, L.TRI_LOWER_UNIT, bw, monkeypatch)[0] == "lsync"
    # a grid launch per level on the same DAG
    with monkeypatch.context() as m:
        m.setenv("RSB_TRSV_GRID", "levels")
        W2 = P.CscMatrix(W.nrows, W.ncols, W.col_ptr.copy(), W.row_idx.copy(), W.values.copy())
        assert check(W2, L.TRI_LOWER_UNIT, bw, monkeypatch)[0] == "levels"


@pytest.mark.parametrize("grid", ["levelsync", "levelsync-n4", "lsync", "syncfree", "syncfree-pairs",
                                  "syncfree-unsorted", "syncfree-n4", "static", "static-n4", "natural",
                                  "natural-cap32", "natural-minb6", "natural-minb8", "natural-static"])
@pytest.mark.parametrize("k", [3, 12, 20])
def test_wide_kernel_every_kind_and_long_tasks(k, grid, monkeypatch):
    """The persistent wide solves (grid schedules): sync-free (the default)
    and level-synchronous.  Tasks past the register entries take the
    out-of-line tail (sequential order); the sync-free kernel waits for it
    without blocking (a dependency may sit in another lane of the warp)."""
    if grid == "lsync":
        monkeypatch.setenv("RSB_TRSV_GRID", "lsync")
    if grid.startswith("levelsync"):
        monkeypatch.setenv("RSB_TRSV_GRID", "levelsync")
    if grid.startswith("static"):
        monkeypatch.setenv("RSB_TRSV_GRID", "static")
    if grid.startswith("syncfree"):
        monkeypatch.setenv("RSB_TRSV_GRID", "syncfree")
    if grid == "static-n4":
        monkeypatch.setenv("RSB_WIDE_N", "4")
    if grid.startswith("natural"):  # index-order kernel (trsv_nat.cu) reading the matrix's own arrays
        monkeypatch.setenv("RSB_TRSV_ORDER", "natural")
    else:
        monkeypatch.setenv("RSB_TRSV_ORDER", "level")
    if grid.endswith("cap32"):  # the smallest window: every slice takes several passes
        monkeypatch.setenv("RSB_NAT_CAP", "32")
    if grid.startswith("natural-minb"):
        monkeypatch.setenv("RSB_NAT_MINB", grid[-1])
    if grid == "natural-static":  # round-robin slices under a cooperative launch instead of the ticket
        monkeypatch.setenv("RSB_NAT_STATIC", "1")
    if grid == "levelsync-n4":  # level-synchronous with 4 register entries: long tasks take the tail
        monkeypatch.setenv("RSB_WIDE_N", "4")
    if grid == "syncfree-pairs":
        monkeypatch.setenv("RSB_WIDE_EARLY", "0")
    if grid == "syncfree-unsorted":
        monkeypatch.setenv("RSB_TRSV_SORT", "0")
    if grid == "syncfree-n4":  # 4 register entries: every longer task takes the batched tail
        monkeypatch.setenv("RSB_WIDE_N", "4")
    rng = np.random.default_rng(100 + k)
    Ms = leveled_lower([5000] * 4, k, rng, window=4000)  # strictly lower: the unit kinds
    b = rng.standard_normal(Ms.ncols)
    for kind in (L.TRI_LOWER_UNIT, L.TRI_LOWER_T_UNIT):
        check(Ms, kind, b, monkeypatch)
    n = Ms.ncols
    cols = np.repeat(np.arange(n), np.diff(Ms.col_ptr))
    M = P.CscMatrix.from_coo(n, n, np.concatenate([Ms.row_idx, np.arange(n)]), np.concatenate([cols, np.arange(n)]),
                             np.concatenate([Ms.values, rng.uniform(1.0, 2.0, n)]))
    for kind in (L.TRI_LOWER, L.TRI_LOWER_T):
        check(M, kind, b, monkeypatch)
    U = transpose(M)
    for kind in (L.TRI_UPPER, L.TRI_UPPER_T):
        check(U, kind, b, monkeypatch)
    want = {"lsync": "lsync", "levelsync": "levelsync", "levelsync-n4": "levelsync"}.get(
        grid, "natural" if grid.startswith("natural") else "grid")
    assert variant(M, L.TRI_LOWER)[0] == want


def test_many_chunks_every_kind(monkeypatch):
    rng = np.random.default_rng(3)
    M = leveled_lower([64] * 700, 8, rng, diag=lambda n: rng.uniform(1.0, 2.0, n) * rng.choice([-1, 1], n))
    b = rng.standard_normal(M.ncols)
    for kind in (L.TRI_LOWER, L.TRI_LOWER_T):
        check(M, kind, b, monkeypatch)
    U = transpose(M)
    for kind in (L.TRI_UPPER, L.TRI_UPPER_T):
        check(U, kind, b, monkeypatch)


def test_division_outside_exact_range(monkeypatch):
    """Diagonals and partial sums outside (2^-500, 2^500), zeros, signed
    zeros, infinities and NaN take IEEE division inside the lean kernel."""
    rng = np.random.default_rng(4)

    def diag(n):
        d = rng.uniform(1.0, 2.0, n)
        d[::7] = 1e-200
        d[3::11] = 1e200
        d[5::13] = -3e-160
        return d

    M = leveled_lower([32] * 90, 4, rng, diag=diag)
    n = M.ncols
    for b in (rng.standard_normal(n), rng.standard_normal(n) * 1e-300, np.zeros(n), -np.zeros(n)):
        check(M, L.TRI_LOWER, b, monkeypatch, ("lean", None))
    b = rng.standard_normal(n)
    b[::17] = 0.0
    b[1::19] = -0.0
    b[2::23] = np.inf
    b[3::29] = np.nan
    b[4::31] = 5e-324
    check(M, L.TRI_LOWER, b, monkeypatch, ("lean", None))
    check(transpose(M), L.TRI_UPPER, b, monkeypatch)


def test_single_level_and_tiny():
    for n in (1, 2, 31, 33):
        M = P.CscMatrix.identity(n)
        b = np.arange(1.0, n + 1.0)
        assert np.array_equal(P.sparse_lower_solve(M, b), b)
        assert np.array_equal(P.sparse_upper_solve(M, b), b)
        E = P.CscMatrix(n, n, np.zeros(n + 1, dtype=np.int64), np.zeros(0, dtype=np.int64), np.zeros(0))
        assert np.array_equal(P.sparse_lower_solve_transpose(E, b, unit_diag=True), b)
        assert np.array_equal(P.sparse_lower_solve(E, b, unit_diag=True), b)
