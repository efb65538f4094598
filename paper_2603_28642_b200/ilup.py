"""Rectangular ILUP factorization (host setup, native C++).

Same parameters, dataclasses and outputs as pkg/src/rowsplit/ilup.py
(IlupParams il.py:27-50, IlupFactors il.py:53-119, ilup_factorize
il.py:211-368); the factorization runs in librowsplit_b200.so
(csrc/host_setup.cpp) and is bit-identical to the reference's (pinned by
tests/test_host_setup.py against factors the reference produced).  It stays
on the CPU: the north star keeps ILUP out of the device path, timed
separately.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from .types import CscMatrix, Permutation


@dataclass
class IlupParams:
    """p: max kept entries per factor column; tau: drop tolerance; mu in (0, 1]:
    pivot threshold (1 = partial pivoting); small: minimum pivot magnitude."""

    p: int = 10
    tau: float = 0.0
    mu: float = 0.1
    small: float = 1e-10

    def __post_init__(self):
        if self.p < 1:
            raise ValueError("p must be >= 1")
        if self.tau < 0.0:
            raise ValueError("tau must be >= 0")
        if not 0.0 < self.mu <= 1.0:
            raise ValueError("mu must be in (0, 1]")
        if self.small <= 0.0:
            raise ValueError("small must be > 0")


@dataclass
class IlupFactors:
    """row_perm maps pivot positions to original rows; L1 n x n unit lower
    (implicit diagonal), L2 the remaining m-n rows, U n x n upper with the
    diagonal stored last in every column."""

    row_perm: Permutation
    L1: CscMatrix
    L2: CscMatrix
    U: CscMatrix
    nmod: int
    row_counts_final: np.ndarray

    @property
    def nrows(self) -> int:
        return self.L1.nrows + self.L2.nrows

    @property
    def ncols(self) -> int:
        return self.U.ncols

    @staticmethod
    def of(f) -> "IlupFactors":
        """Adopt a reference IlupFactors (or anything shaped like one)."""
        if isinstance(f, IlupFactors):
            return f
        rp = f.row_perm
        return IlupFactors(Permutation(np.asarray(rp.perm), np.asarray(rp.inv)), CscMatrix.of(f.L1),
                           CscMatrix.of(f.L2), CscMatrix.of(f.U), int(f.nmod),
                           np.asarray(f.row_counts_final))


def ilup_factorize(A, params: IlupParams | None = None) -> IlupFactors:
    """Incomplete LU with threshold pivoting of an m x n (m >= n) matrix."""
    params = params or IlupParams()
    m, n = int(A.nrows), int(A.ncols)
    if n < 1 or m < 1:
        raise ValueError("empty matrix")
    if m < n:
        raise ValueError(f"need nrows >= ncols, got {m} x {n}")
    cp, ri, va = L.i64c(A.col_ptr), L.i64c(A.row_idx), L.f64c(A.values)
    h = ctypes.c_void_p()
    L.check(L.lib().rsb_ilup_factorize(m, n, L.ptr(cp), L.ptr(ri), L.ptr(va), int(params.p),
                                       float(params.tau), float(params.mu), float(params.small),
                                       ctypes.byref(h)))
    try:
        n1, n2, nu, nmod = (ctypes.c_int64() for _ in range(4))
        L.check(L.lib().rsb_ilup_sizes(h, ctypes.byref(n1), ctypes.byref(n2), ctypes.byref(nu),
                                       ctypes.byref(nmod)))
        perm = np.empty(m, dtype=np.int64)
        l1p, l2p, up = (np.empty(n + 1, dtype=np.int64) for _ in range(3))
        l1i, l1v = np.empty(max(1, n1.value), dtype=np.int64), np.empty(max(1, n1.value))
        l2i, l2v = np.empty(max(1, n2.value), dtype=np.int64), np.empty(max(1, n2.value))
        ui, uv = np.empty(max(1, nu.value), dtype=np.int64), np.empty(max(1, nu.value))
        rc = np.empty(m, dtype=np.int64)
        L.check(L.lib().rsb_ilup_copy(h, L.ptr(perm), L.ptr(l1p), L.ptr(l1i), L.ptr(l1v), L.ptr(l2p),
                                      L.ptr(l2i), L.ptr(l2v), L.ptr(up), L.ptr(ui), L.ptr(uv), L.ptr(rc)))
    finally:
        L.lib().rsb_ilup_destroy(h)
    k1, k2, ku = n1.value, n2.value, nu.value
    return IlupFactors(
        row_perm=Permutation.from_perm(perm),
        L1=CscMatrix(n, n, l1p, l1i[:k1], l1v[:k1]),
        L2=CscMatrix(m - n, n, l2p, l2i[:k2], l2v[:k2]),
        U=CscMatrix(n, n, up, ui[:ku], uv[:ku]),
        nmod=int(nmod.value),
        row_counts_final=rc,
    )
