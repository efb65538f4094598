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


# ---------------------------------------------------------------------------
# on-disk factor cache (host setup is the slow part of a config-4 run: the
# serial ILUP takes minutes at n = 8e6)
# ---------------------------------------------------------------------------

_FACTOR_FIELDS = ("perm", "L1_ptr", "L1_idx", "L1_val", "L2_ptr", "L2_idx", "L2_val", "U_ptr", "U_idx",
                  "U_val", "row_counts")


def _cache_key(A, params: IlupParams) -> str:
    import hashlib

    h = hashlib.sha256()
    h.update(f"{int(A.nrows)}x{int(A.ncols)}|p={params.p}|tau={params.tau!r}|mu={params.mu!r}|"
             f"small={params.small!r}|v2".encode())
    for a in (A.col_ptr, A.row_idx, A.values):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:24]


def ilup_factorize_cached(A, params: IlupParams | None = None, cache_dir: str | None = None) -> IlupFactors:
    """ilup_factorize with an on-disk cache keyed by a digest of A and the
    parameters (cache_dir, else $RSB_FACTOR_CACHE; no caching when neither is
    set).  A hit returns the stored factors unchanged: the same bits the
    factorization produces."""
    import os

    params = params or IlupParams()
    cache_dir = cache_dir or os.environ.get("RSB_FACTOR_CACHE")
    if not cache_dir:
        return ilup_factorize(A, params)
    d = os.path.join(cache_dir, "ilup_" + _cache_key(A, params))
    m, n = int(A.nrows), int(A.ncols)
    try:
        z = {k: np.load(os.path.join(d, k + ".npy")) for k in _FACTOR_FIELDS}
        meta = np.load(os.path.join(d, "meta.npy"))
        return IlupFactors(
            row_perm=Permutation.from_perm(z["perm"]),
            L1=CscMatrix(n, n, z["L1_ptr"], z["L1_idx"], z["L1_val"]),
            L2=CscMatrix(m - n, n, z["L2_ptr"], z["L2_idx"], z["L2_val"]),
            U=CscMatrix(n, n, z["U_ptr"], z["U_idx"], z["U_val"]),
            nmod=int(meta[0]), row_counts_final=z["row_counts"])
    except (OSError, ValueError, KeyError):
        pass
    f = ilup_factorize(A, params)
    tmp = d + f".tmp{os.getpid()}"
    os.makedirs(tmp, exist_ok=True)
    arrays = {"perm": f.row_perm.perm, "row_counts": f.row_counts_final}
    for k in ("L1", "L2", "U"):
        M = getattr(f, k)
        arrays.update({f"{k}_ptr": M.col_ptr, f"{k}_idx": M.row_idx, f"{k}_val": M.values})
    for k, v in arrays.items():
        np.save(os.path.join(tmp, k + ".npy"), np.ascontiguousarray(v))
    np.save(os.path.join(tmp, "meta.npy"), np.array([f.nmod], dtype=np.int64))
    try:
        os.replace(tmp, d)
    except OSError:
        pass
    return f
