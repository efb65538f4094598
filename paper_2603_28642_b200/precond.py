"""Row-splitting preconditioner with the reference's API, applied on the B200.

Mirrors pkg/src/rowsplit/precond.py (pc.py): SMode/YMode (pc.py:36-48),
RowSplitPreconditioner (pc.py:106-186) and build_preconditioner
(pc.py:323-362).  Construction (explicit Y, the dense coupling matrix and
its Cholesky factor) is host setup; every application -- apply, y_apply,
y_apply_transpose, s_matvec_implicit -- runs as sm_100a kernels
(csrc/solver.cu enqueue_apply) with results bit-identical to the reference.
"""

from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .device import device_preconditioner
from .ilup import IlupFactors
from .sparse import dense_cholesky_factorize
from .types import CscMatrix, DenseMatrix


class SMode(enum.Enum):
    """How the coupling system S w = u is solved (pc.py:36-41)."""

    DENSE_FACTOR = "dense"
    INNER_CG = "cg"
    IDENTITY = "identity"


class YMode(enum.Enum):
    """Y = L2 L1^{-1} stored, or applied through solves (pc.py:44-48)."""

    EXPLICIT = "explicit"
    IMPLICIT = "implicit"


def _smode(m) -> SMode:
    return m if isinstance(m, SMode) else SMode(getattr(m, "value", m))


def _ymode(m) -> YMode | None:
    if m is None:
        return None
    return m if isinstance(m, YMode) else YMode(getattr(m, "value", m))


def build_y_explicit(factors) -> CscMatrix:
    """Y = L2 L1^{-1} as a sparse (m-n) x n matrix (pc.py:55-82), host native."""
    L1, L2 = factors.L1, factors.L2
    s, n = int(L2.nrows), int(L2.ncols)
    a = [L.i64c(L1.col_ptr), L.i64c(L1.row_idx), L.f64c(L1.values),
         L.i64c(L2.col_ptr), L.i64c(L2.row_idx), L.f64c(L2.values)]
    nnz = ctypes.c_int64(0)
    args = [L.ptr(v) for v in a]
    L.check(L.lib().rsb_build_y_explicit(s, n, *args, ctypes.byref(nnz), None, None, None))
    yp = np.empty(n + 1, dtype=np.int64)
    yi = np.empty(max(1, nnz.value), dtype=np.int64)
    yv = np.empty(max(1, nnz.value))
    L.check(L.lib().rsb_build_y_explicit(s, n, *args, ctypes.byref(nnz), L.ptr(yp), L.ptr(yi), L.ptr(yv)))
    k = nnz.value
    return CscMatrix(s, n, yp, yi[:k], yv[:k])


def _setup_where(setup) -> str:
    where = setup if setup is not None else os.environ.get("RSB_SETUP", "host")
    if where not in ("host", "device"):
        raise ValueError("setup must be 'host' or 'device'")
    return where


def dense_build_device(factors, what: int = 1):
    """Y = L2 L1^{-1}, S = I + Y Y^T and its Cholesky factor, formed on the
    device (csrc/dbuild.cu; pc.py:55-103, sc.py:585-604).

    what = 0: Y only; 1: Y and the S factor; 2: also S.  Returns (Y,
    S or None, S_factor or None, seconds of the three phases).  Y and the
    factor-given-S are bit-identical to the reference; S is a fixed-order
    FP64 product within rounding of numpy's ``yd @ yd.T``.
    """
    from .device import device_matrix, get_context

    factors = IlupFactors.of(factors)
    ctx = get_context()
    d1, d2 = device_matrix(factors.L1, ctx), device_matrix(factors.L2, ctx)
    h = ctypes.c_void_p()
    L.check(L.lib().rsb_dense_build(d1.h, d2.h, int(what), ctypes.byref(h)))
    try:
        s, n, nnz = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        sec = np.zeros(3)
        L.check(L.lib().rsb_dense_build_sizes(h, ctypes.byref(s), ctypes.byref(n), ctypes.byref(nnz),
                                              sec.ctypes.data_as(L.f64p)))
        s, n, k = s.value, n.value, nnz.value
        yp = np.empty(n + 1, dtype=np.int64)
        yi = np.empty(max(1, k), dtype=np.int64)
        yv = np.empty(max(1, k))
        S = np.empty((s, s), order="F") if what == 2 else None
        F = np.empty((s, s), order="F") if what >= 1 else None
        L.check(L.lib().rsb_dense_build_copy(
            h, L.ptr(yp), L.ptr(yi), L.ptr(yv),
            L.ptr(S.ravel(order="K")) if S is not None and s else None,
            L.ptr(F.ravel(order="K")) if F is not None and s else None))
    finally:
        L.lib().rsb_dense_build_destroy(h)
    Y = CscMatrix(s, n, yp, yi[:k], yv[:k])
    return (Y, DenseMatrix(S) if S is not None else None, DenseMatrix(F) if F is not None else None,
            tuple(float(v) for v in sec))


def _gram_plus_identity(Y) -> DenseMatrix:
    """I + Y Y^T with the lower triangle mirrored (pc.py:85-92).  Host BLAS,
    the same dense product the reference forms."""
    yd = CscMatrix.of(Y).to_dense()
    g = yd @ yd.T
    s = np.asfortranarray(np.tril(g) + np.tril(g, -1).T)
    s[np.arange(Y.nrows), np.arange(Y.nrows)] += 1.0
    return DenseMatrix(s)


def assemble_s_dense(pre) -> DenseMatrix:
    """Dense coupling matrix I + Y Y^T of a built preconditioner (pc.py:95-103)."""
    if pre.Y is None:
        raise ValueError("dense assembly needs the explicit Y")
    if pre.Y.nrows > pre.dense_cap:
        raise ValueError(f"coupling block of size {pre.Y.nrows} exceeds the dense cap {pre.dense_cap}")
    return _gram_plus_identity(pre.Y)


def _psize(factors, Y, S_factor) -> int:
    size = factors.L1.nnz + factors.L2.nnz + factors.U.nnz
    if Y is not None:
        size += Y.nnz
    if S_factor is not None:
        s = S_factor.nrows
        size += s * (s + 1) // 2
    return size


@dataclass
class RowSplitPreconditioner:
    """Applied form of the row-splitting preconditioner (pc.py:106-186).

    Immutable once built.  Applications run on the device; the device copy
    of the factors is made on first use and cached.
    """

    factors: IlupFactors
    y_mode: YMode
    s_mode: SMode
    cg_iters: int
    Y: CscMatrix | None
    S_factor: DenseMatrix | None
    psize: int
    dense_cap: int

    @property
    def n(self) -> int:
        return self.factors.ncols

    @property
    def split_rows(self) -> int:
        return self.factors.L2.nrows

    def _dev(self):
        return device_preconditioner(self)

    def y_apply(self, r1):
        """Y @ r1 (pc.py:135-139)."""
        return self._dev().y_apply(r1)

    def y_apply_transpose(self, w):
        """Y.T @ w (pc.py:141-147)."""
        return self._dev().y_apply_transpose(w)

    def s_matvec_implicit(self, v):
        """(I + L2 L1^{-1} L1^{-T} L2^T) v without forming Y (pc.py:149-154)."""
        return self._dev().s_matvec(v)

    def apply(self, r1, r2) -> np.ndarray:
        """h with L1 U h = r1 + Y^T w, S w = r2 - Y r1 (pc.py:167-186)."""
        r1 = np.asarray(r1, dtype=np.float64)
        r2 = np.asarray(r2, dtype=np.float64)
        if r1.shape != (self.n,) or r2.shape != (self.split_rows,):
            raise ValueError("residual component lengths do not match the split")
        return self._dev().apply(r1, r2)


def build_preconditioner(
    factors,
    s_mode: SMode = SMode.DENSE_FACTOR,
    y_mode: YMode | None = None,
    cg_iters: int = 2,
    dense_cap: int = 20000,
    *,
    setup: str | None = None,
) -> RowSplitPreconditioner:
    """Assemble the applied preconditioner (pc.py:323-362).

    y_mode defaults to explicit for the dense S factorization and implicit
    otherwise; ValueError for a dense request above dense_cap.  setup
    ('host', default, or 'device'; env RSB_SETUP) says where the explicit Y,
    S = I + Y Y^T and its Cholesky factor are formed: the host build is
    bit-identical to the reference throughout; the device build
    (dense_build_device) gives the same Y bits and the same factor bits for
    a given S, with S itself within rounding of the reference's BLAS product.
    """
    where = _setup_where(setup)
    factors = IlupFactors.of(factors)
    s_mode = _smode(s_mode)
    y_mode = _ymode(y_mode)
    if cg_iters < 1:
        raise ValueError("cg_iters must be >= 1")
    if y_mode is None:
        y_mode = YMode.EXPLICIT if s_mode is SMode.DENSE_FACTOR else YMode.IMPLICIT
    if s_mode is SMode.DENSE_FACTOR and y_mode is not YMode.EXPLICIT:
        raise ValueError("dense S factorization requires the explicit Y")
    s = factors.L2.nrows
    if s_mode is SMode.DENSE_FACTOR and s > dense_cap:
        raise ValueError(f"coupling block of size {s} exceeds the dense cap {dense_cap}")
    Y = S_factor = None
    if y_mode is YMode.EXPLICIT and where == "device":
        Y, _, S_factor, _ = dense_build_device(factors, 1 if s_mode is SMode.DENSE_FACTOR else 0)
    elif y_mode is YMode.EXPLICIT:
        Y = build_y_explicit(factors)
        if s_mode is SMode.DENSE_FACTOR:
            S_factor = dense_cholesky_factorize(_gram_plus_identity(Y))
    return RowSplitPreconditioner(
        factors=factors, y_mode=y_mode, s_mode=s_mode, cg_iters=cg_iters, Y=Y,
        S_factor=S_factor, psize=_psize(factors, Y, S_factor), dense_cap=dense_cap,
    )
