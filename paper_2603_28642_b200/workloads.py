"""Seeded synthetic inputs for the five BASELINE.json configurations.

No public dataset is named by BASELINE.json; these generators stand in for
the problems it describes (shapes, sparsity and value distributions from
BASELINE.json ``configs`` and SURVEY.md section 8(d)).  Seed = config index
unless given.  The order of RNG draws is part of the definition and is
listed in each docstring, so a generator gives the same matrix on every
host (numpy's PCG64 + the distribution algorithms are platform-stable).

Each generator returns (A, rhs) where A is a CscMatrix (sorted rows, no
stored zeros, duplicates summed -- the reference's CscMatrix.from_coo
contract, sparse_core.py:84-106) and rhs is a float64 array of shape (m,)
or (nrhs, m).
"""

from __future__ import annotations

import numpy as np

from .types import CscMatrix


def _stacked_random_rows(rng, m, n, k_top_off, k_bottom, diag=True):
    """Rows 0..n-1: diagonal +-U(1,2) plus k_top_off N(0,1) entries at uniform
    columns; rows n..m-1: k_bottom N(0,1) entries at uniform columns.

    Draw order: sign (n), magnitude (n), top columns (n, k_top_off),
    top values (n, k_top_off), bottom columns (m-n, k_bottom), bottom values.
    """
    sign = rng.choice(np.array([-1.0, 1.0]), size=n)
    mag = rng.uniform(1.0, 2.0, size=n)
    tcols = rng.integers(0, n, size=(n, k_top_off))
    tvals = rng.standard_normal((n, k_top_off))
    bcols = rng.integers(0, n, size=(m - n, k_bottom))
    bvals = rng.standard_normal((m - n, k_bottom))
    top_rows = np.repeat(np.arange(n, dtype=np.int64), k_top_off)
    bot_rows = np.repeat(np.arange(n, m, dtype=np.int64), k_bottom)
    rows = [top_rows, bot_rows]
    cols = [tcols.ravel(), bcols.ravel()]
    vals = [tvals.ravel(), bvals.ravel()]
    if diag:
        rows.insert(0, np.arange(n, dtype=np.int64))
        cols.insert(0, np.arange(n, dtype=np.int64))
        vals.insert(0, sign * mag)
    return np.concatenate(rows), np.concatenate(cols), np.concatenate(vals)


def config0(seed=0, m=3000, n=2000):
    """m=3000, n=2000: rows 0..n-1 diagonal +-U(1,2) + 3 N(0,1) off-diagonals,
    rows n..m-1 five N(0,1) entries; rows permuted; b ~ N(0,1)^m.

    Draws: _stacked_random_rows(k_top_off=3, k_bottom=5), permutation(m), b.
    """
    rng = np.random.default_rng(seed)
    r, c, v = _stacked_random_rows(rng, m, n, 3, 5)
    perm = rng.permutation(m)
    A = CscMatrix.from_coo(m, n, perm[r], c, v)
    b = rng.standard_normal(m)
    return A, b


def config1(seed=1, g=256, n_obs=None, obs_k=8):
    """Overdetermined 2-D grid problem: n = g*g unknowns, 5-point Laplacian
    (4 + 0.01 on the diagonal, -1 to in-grid neighbours, Dirichlet), then
    n_obs = n/2 observation rows with obs_k uniform columns and U(0,1)
    weights normalised to sum 1; b = A x_true + 1e-3 N(0,1), x_true ~ N(0,1).

    Draws: observation columns (n_obs, obs_k), weights (n_obs, obs_k),
    x_true (n), noise (m).
    """
    rng = np.random.default_rng(seed)
    n = g * g
    n_obs = n // 2 if n_obs is None else n_obs
    m = n + n_obs
    idx = np.arange(n, dtype=np.int64)
    gi, gj = idx // g, idx % g
    rows = [idx]
    cols = [idx]
    vals = [np.full(n, 4.01)]
    for di, dj in ((-1, 0), (1, 0), (0, -1), (0, 1)):
        ok = (gi + di >= 0) & (gi + di < g) & (gj + dj >= 0) & (gj + dj < g)
        rows.append(idx[ok])
        cols.append((gi[ok] + di) * g + gj[ok] + dj)
        vals.append(np.full(int(ok.sum()), -1.0))
    ocols = rng.integers(0, n, size=(n_obs, obs_k))
    w = rng.uniform(0.0, 1.0, size=(n_obs, obs_k))
    w = w / w.sum(axis=1, keepdims=True)
    rows.append(np.repeat(np.arange(n, m, dtype=np.int64), obs_k))
    cols.append(ocols.ravel())
    vals.append(w.ravel())
    A = CscMatrix.from_coo(m, n, np.concatenate(rows), np.concatenate(cols), np.concatenate(vals))
    x_true = rng.standard_normal(n)
    noise = rng.standard_normal(m)
    b = _host_matvec(A, x_true) + 1e-3 * noise
    return A, b


def config2(seed=2, n=100_000, s=100, density=0.5):
    """Sparse-dense problem: n rows as config 0 with 6 nnz/row (diagonal + 5
    off-diagonals), plus s dense rows where each column is present with
    probability `density`, values N(0,1)/sqrt(n); rows permuted; b ~ N(0,1).

    Draws: _stacked_random_rows(k_top_off=5, k_bottom=0), dense mask (s, n),
    dense values (s, n), permutation(m), b.
    """
    rng = np.random.default_rng(seed)
    m = n + s
    r, c, v = _stacked_random_rows(rng, n, n, 5, 0)
    mask = rng.random((s, n)) < density
    dv = rng.standard_normal((s, n)) / np.sqrt(n)
    dr, dc = np.nonzero(mask)
    rows = np.concatenate([r, n + dr.astype(np.int64)])
    cols = np.concatenate([c, dc.astype(np.int64)])
    vals = np.concatenate([v, dv[dr, dc]])
    perm = rng.permutation(m)
    A = CscMatrix.from_coo(m, n, perm[rows], cols, vals)
    b = rng.standard_normal(m)
    return A, b


def config3(seed=3, n=1_000_000, m=None, k=8):
    """Ill-conditioned sparse problem: m = 1.5 n rows with k uniform N(0,1)
    entries each, plus a +-U(1,2) entry at (sel_j, j) for n distinct randomly
    chosen rows sel; columns then scaled by 10^U(-4,4).  Run unscaled.

    Draws: columns (m, k), values (m, k), sel = permutation(m)[:n],
    sign (n), magnitude (n), column exponents (n), b.
    """
    rng = np.random.default_rng(seed)
    m = (3 * n) // 2 if m is None else m
    cols = rng.integers(0, n, size=(m, k))
    vals = rng.standard_normal((m, k))
    sel = rng.permutation(m)[:n]
    sign = rng.choice(np.array([-1.0, 1.0]), size=n)
    mag = rng.uniform(1.0, 2.0, size=n)
    expo = rng.uniform(-4.0, 4.0, size=n)
    rows = np.concatenate([np.repeat(np.arange(m, dtype=np.int64), k), sel.astype(np.int64)])
    cc = np.concatenate([cols.ravel(), np.arange(n, dtype=np.int64)])
    vv = np.concatenate([vals.ravel(), sign * mag])
    vv = vv * (10.0 ** expo)[cc]
    A = CscMatrix.from_coo(m, n, rows, cc, vv)
    b = rng.standard_normal(m)
    return A, b


def config4(seed=4, n=8_000_000, m=None, nrhs=64, first_rhs=0):
    """Multi-GPU scale problem: as config 0 with 6 nnz/row -- rows 0..n-1
    diagonal + 5 off-diagonals, rows n..m-1 six N(0,1) entries, m = 2n; rows
    permuted; right-hand sides N(0,1)^m drawn in order.  Returns the rhs
    j = first_rhs .. first_rhs + nrhs - 1 of that sequence (the earlier
    ones are drawn and discarded), so a rank's shard of the 64-RHS batch is
    the same vectors whichever rank draws it.

    Draws: _stacked_random_rows(k_top_off=5, k_bottom=6), permutation(m),
    then rhs j = 0, 1, ... each standard_normal(m).
    """
    rng = np.random.default_rng(seed)
    m = 2 * n if m is None else m
    r, c, v = _stacked_random_rows(rng, m, n, 5, 6)
    perm = rng.permutation(m)
    A = CscMatrix.from_coo(m, n, perm[r], c, v)
    del r, c, v, perm
    for _ in range(first_rhs):
        rng.standard_normal(m)
    B = np.empty((nrhs, m))
    for j in range(nrhs):
        B[j] = rng.standard_normal(m)
    return A, B


def _host_matvec(A, x):
    """y = A x in the reference's scatter order (input generation only)."""
    y = np.zeros(A.nrows)
    if A.nnz:
        np.add.at(y, A.row_idx, A.values * np.repeat(x, A.column_counts()))
    return y


GENERATORS = {0: config0, 1: config1, 2: config2, 3: config3, 4: config4}

# Solver / factorization settings per config.
SETTINGS = {
    0: dict(p=10, tau=1e-3, delta=1e-8, max_iters=2000, scale=True, s_mode="dense"),
    1: dict(p=10, tau=0.0, delta=1e-10, max_iters=2000, scale=True, s_mode="cg"),
    2: dict(p=10, tau=0.0, delta=1e-8, max_iters=2000, scale=True, s_mode="dense"),
    3: dict(p=10, tau=0.0, delta=1e-8, max_iters=20000, scale=False, s_mode="cg"),
    4: dict(p=10, tau=0.0, delta=1e-8, max_iters=2000, scale=True, s_mode="cg"),
}
