"""Host-side data types consumed by the B200 solve path.

They mirror the reference's types field for field (sparse_core.py:27-204:
CscMatrix, DenseMatrix, Permutation, ColumnScaling) so factors, matrices
and vectors move between the two packages unchanged; any object with the
same attributes (e.g. a reference CscMatrix) is accepted wherever these
are.  All values are float64 and all index arrays int64 on the host; the
device copies use int32 indices ("Data layout in HBM").
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class CscMatrix:
    """Compressed sparse column matrix: rows strictly increasing within a
    column, no stored zeros (reference contract, sparse_core.py:27-33)."""

    __slots__ = ("nrows", "ncols", "col_ptr", "row_idx", "values", "_dev")

    def __init__(self, nrows, ncols, col_ptr, row_idx, values):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int64)
        self.row_idx = np.ascontiguousarray(row_idx, dtype=np.int64)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self._dev = None

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])

    def column(self, j):
        lo, hi = self.col_ptr[j], self.col_ptr[j + 1]
        return self.row_idx[lo:hi], self.values[lo:hi]

    def column_counts(self):
        return np.diff(self.col_ptr)

    def validate(self):
        """Structural invariants (reference sparse_core.py:56-82); ValueError."""
        if self.nrows < 0 or self.ncols < 0:
            raise ValueError("negative dimension")
        if self.col_ptr.shape != (self.ncols + 1,):
            raise ValueError("col_ptr has wrong length")
        if self.col_ptr[0] != 0 or self.col_ptr[-1] != len(self.row_idx):
            raise ValueError("col_ptr endpoints inconsistent with storage")
        counts = np.diff(self.col_ptr)
        if np.any(counts < 0):
            raise ValueError("col_ptr not non-decreasing")
        if len(self.row_idx) != len(self.values):
            raise ValueError("row_idx and values length mismatch")
        if self.nnz:
            if self.row_idx.min() < 0 or self.row_idx.max() >= self.nrows:
                raise ValueError("row index out of range")
            if np.any(self.values == 0.0):
                raise ValueError("explicitly stored zero")
            # strictly increasing inside every column: compare neighbours that
            # share a column
            same_col = np.repeat(np.arange(self.ncols), counts)
            inner = same_col[1:] == same_col[:-1]
            if np.any(np.diff(self.row_idx)[inner] <= 0):
                raise ValueError("row indices not strictly increasing in a column")
        return self

    @staticmethod
    def from_coo(nrows, ncols, rows, cols, vals):
        """Triplets -> CSC; duplicates summed in input order, zeros dropped."""
        rows = np.asarray(rows, dtype=np.int64).ravel()
        cols = np.asarray(cols, dtype=np.int64).ravel()
        vals = np.asarray(vals, dtype=np.float64).ravel()
        nrows, ncols = int(nrows), int(ncols)
        if len(rows):
            key = cols * max(nrows, 1) + rows
            order = np.argsort(key, kind="stable")
            key, rows, cols, vals = key[order], rows[order], cols[order], vals[order]
            head = np.ones(len(key), dtype=bool)
            head[1:] = key[1:] != key[:-1]
            if not head.all():
                run = np.cumsum(head) - 1
                acc = np.zeros(int(run[-1]) + 1)
                np.add.at(acc, run, vals)
                rows, cols, vals = rows[head], cols[head], acc
            nz = vals != 0.0
            if not nz.all():
                rows, cols, vals = rows[nz], cols[nz], vals[nz]
        col_ptr = np.zeros(ncols + 1, dtype=np.int64)
        if len(cols):
            col_ptr[1:] = np.cumsum(np.bincount(cols, minlength=ncols))
        return CscMatrix(nrows, ncols, col_ptr, rows, vals)

    @staticmethod
    def from_dense(a, drop_below=0.0):
        a = np.asarray(a, dtype=np.float64)
        r, c = np.nonzero(np.abs(a) > drop_below)
        return CscMatrix.from_coo(a.shape[0], a.shape[1], r, c, a[r, c])

    @staticmethod
    def identity(n):
        i = np.arange(n, dtype=np.int64)
        return CscMatrix(n, n, np.arange(n + 1, dtype=np.int64), i, np.ones(n))

    @staticmethod
    def of(M) -> "CscMatrix":
        """Adopt any CSC-shaped object (e.g. a reference CscMatrix)."""
        if isinstance(M, CscMatrix):
            return M
        return CscMatrix(M.nrows, M.ncols, M.col_ptr, M.row_idx, M.values)

    def to_dense(self):
        out = np.zeros((self.nrows, self.ncols))
        if self.nnz:
            out[self.row_idx, np.repeat(np.arange(self.ncols), self.column_counts())] = self.values
        return out

    def transpose(self) -> "CscMatrix":
        c = np.repeat(np.arange(self.ncols, dtype=np.int64), self.column_counts())
        return CscMatrix.from_coo(self.ncols, self.nrows, c, self.row_idx, self.values)

    def __repr__(self):
        return f"CscMatrix({self.nrows}x{self.ncols}, nnz={self.nnz})"


class DenseMatrix:
    """Small dense matrix in column-major order (sparse_core.py:134-158)."""

    __slots__ = ("a",)

    def __init__(self, a):
        self.a = np.asfortranarray(a, dtype=np.float64)
        if self.a.ndim != 2:
            raise ValueError("DenseMatrix expects a 2-d array")

    @property
    def nrows(self):
        return self.a.shape[0]

    @property
    def ncols(self):
        return self.a.shape[1]

    @property
    def values(self):
        return self.a.ravel(order="F")


@dataclass
class Permutation:
    """perm[i] = original row placed at pivot position i (sparse_core.py:161-193)."""

    perm: np.ndarray
    inv: np.ndarray

    @staticmethod
    def identity(n):
        i = np.arange(n, dtype=np.int64)
        return Permutation(i, i.copy())

    @staticmethod
    def from_perm(perm):
        perm = np.asarray(perm, dtype=np.int64)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(len(perm), dtype=np.int64)
        return Permutation(perm, inv)

    def validate(self):
        if len(self.inv) != len(self.perm):
            raise ValueError("perm/inv length mismatch")
        if not np.array_equal(self.perm[self.inv], np.arange(len(self.perm))):
            raise ValueError("perm and inv are not mutually inverse")
        return self

    def apply(self, v):
        return np.asarray(v)[self.perm]

    def apply_inverse(self, v):
        return np.asarray(v)[self.inv]


@dataclass
class ColumnScaling:
    """Column norms removed by column_scale (sparse_core.py:196-204)."""

    scale: np.ndarray

    def unscale_solution(self, y):
        return np.asarray(y) / self.scale
