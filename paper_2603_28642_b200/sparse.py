"""Sparse kernels with the reference's signatures, run on the B200.

Mirrors pkg/src/rowsplit/sparse_core.py (sc.py): matvec (sc.py:212),
matvec_transpose (sc.py:224), the four triangular solves (sc.py:243-313),
power_method_norm2 (sc.py:428), dense_cholesky_solve (sc.py:607) execute as
sm_100a kernels through librowsplit_b200.so; column_scale (sc.py:405) and
dense_cholesky_factorize (sc.py:585) are native host setup.  Same argument
meaning, same exceptions (ValueError / numpy.linalg.LinAlgError), results
bit-identical to the reference's.
"""

from __future__ import annotations

import os

import numpy as np

from . import _lib as L
from .device import device_matrix, get_context
from .types import ColumnScaling, CscMatrix, DenseMatrix


def _vec(v, n, what):
    v = np.asarray(v, dtype=np.float64)
    if v.shape != (n,):
        raise ValueError(f"{what} has length {v.shape}, expected ({n},)")
    return np.ascontiguousarray(v)


def matvec(A, x) -> np.ndarray:
    """A @ x (sc.py:212-221)."""
    x = _vec(x, int(A.ncols), "x")
    y = np.empty(int(A.nrows))
    if len(y):
        L.check(L.lib().rsb_matvec(device_matrix(A).h, L.ptr(x), L.ptr(y), L.RSB_HOST))
    return y


def matvec_transpose(A, y) -> np.ndarray:
    """A.T @ y (sc.py:224-235)."""
    y = _vec(y, int(A.nrows), "y")
    z = np.empty(int(A.ncols))
    if len(z):
        L.check(L.lib().rsb_matvec_transpose(device_matrix(A).h, L.ptr(y), L.ptr(z), L.RSB_HOST))
    return z


def _check_square(T, b):
    if int(T.nrows) != int(T.ncols):
        raise ValueError("triangular solve needs a square matrix")
    if np.shape(b) != (int(T.ncols),):
        raise ValueError("right-hand side length mismatch")


def _trsv(T, b, kind):
    _check_square(T, b)
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty(len(b))
    if len(b):
        L.check(L.lib().rsb_trsv(device_matrix(T).h, kind, L.ptr(b), L.ptr(x), L.RSB_HOST))
    return x


def sparse_lower_solve(L_, b, unit_diag=False) -> np.ndarray:
    """Forward substitution (sc.py:243-263)."""
    return _trsv(L_, b, L.TRI_LOWER_UNIT if unit_diag else L.TRI_LOWER)


def sparse_upper_solve(U, b) -> np.ndarray:
    """Back substitution, diagonal stored last (sc.py:266-279)."""
    return _trsv(U, b, L.TRI_UPPER)


def sparse_lower_solve_transpose(L_, b, unit_diag=False) -> np.ndarray:
    """L.T x = b from L's storage (sc.py:282-298)."""
    return _trsv(L_, b, L.TRI_LOWER_T_UNIT if unit_diag else L.TRI_LOWER_T)


def sparse_upper_solve_transpose(U, b) -> np.ndarray:
    """U.T x = b from U's storage (sc.py:301-313)."""
    return _trsv(U, b, L.TRI_UPPER_T)


def triangular_levels(T, kind) -> tuple[int, int]:
    """(dependency levels, widest level) of a triangular solve's DAG."""
    return device_matrix(T).levels(kind)


def power_method_norm2(A, iters=100, seed=0) -> float:
    """Spectral-norm estimate by power iteration on A.T A (sc.py:428-454).

    The starting vector is drawn on the host exactly as the reference does
    (numpy default_rng(seed).standard_normal); the 2*iters products run on
    the device.
    """
    if iters < 1:
        raise ValueError("iters must be >= 1")
    v0 = np.random.default_rng(seed).standard_normal(int(A.ncols))
    if int(A.ncols) == 0:
        return 0.0
    est = np.zeros(1)
    L.check(L.lib().rsb_power_norm2(device_matrix(A).h, L.ptr(v0), int(iters),
                                    est.ctypes.data_as(L.f64p)))
    return float(est[0])


def column_scale(A, *, setup: str | None = None):
    """Scale every column of A to unit 2-norm (sc.py:405-425), bit-identical.
    setup='host' (default; env RSB_SETUP) runs the native host loop,
    'device' one kernel (csrc/dbuild.cu k_colscale: the same per-column
    p0 + pairwise order, IEEE sqrt and divide)."""
    where = setup if setup is not None else os.environ.get("RSB_SETUP", "host")
    if where not in ("host", "device"):
        raise ValueError("setup must be 'host' or 'device'")
    cp = L.i64c(A.col_ptr)
    counts = np.diff(cp)
    empty = np.flatnonzero(counts == 0)
    if len(empty):
        raise ValueError(f"cannot scale zero column {empty[0]}")
    vals = L.f64c(A.values)
    scaled = np.empty_like(vals)
    norms = np.empty(int(A.ncols))
    if where == "device":
        L.check(L.lib().rsb_column_scale_device(get_context().h, int(A.ncols), L.ptr(cp), L.ptr(vals), L.ptr(scaled),
                                                L.ptr(norms)))
    else:
        L.check(L.lib().rsb_column_scale(int(A.ncols), L.ptr(cp), L.ptr(vals), L.ptr(scaled), L.ptr(norms)))
    out = CscMatrix(A.nrows, A.ncols, cp.copy(), L.i64c(A.row_idx).copy(), scaled)
    return out, ColumnScaling(norms)


def dense_cholesky_factorize(S, *, setup: str | None = None) -> DenseMatrix:
    """Lower Cholesky factor (sc.py:585-604), bit-identical.  setup='host'
    (default; env RSB_SETUP) runs the native host sweep, 'device' the
    blocked right-looking kernels of csrc/dbuild.cu (same per-element
    subtraction order)."""
    a = getattr(S, "a", S)
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise ValueError("Cholesky needs a square matrix")
    g = np.array(a, order="F", copy=True)
    where = setup if setup is not None else os.environ.get("RSB_SETUP", "host")
    if where == "device":
        L.check(L.lib().rsb_cholesky_factorize_device(get_context().h, g.shape[0], L.ptr(g.ravel(order="K")),
                                                      L.RSB_HOST))
    elif where == "host":
        L.check(L.lib().rsb_cholesky_factorize(g.shape[0], L.ptr(g.ravel(order="K"))))
    else:
        raise ValueError("setup must be 'host' or 'device'")
    return DenseMatrix(g)


def dense_cholesky_solve(factor, b) -> np.ndarray:
    """S x = b given the lower Cholesky factor (sc.py:607-622), on the device."""
    g = np.asfortranarray(getattr(factor, "a", factor), dtype=np.float64)
    s = g.shape[0]
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (s,):
        raise ValueError("right-hand side length mismatch")
    b = np.ascontiguousarray(b)
    x = np.empty(s)
    if s:
        L.check(L.lib().rsb_chol_solve(get_context().h, s, L.ptr(g.ravel(order="F")), L.ptr(b),
                                       L.ptr(x), L.RSB_HOST))
    return x
