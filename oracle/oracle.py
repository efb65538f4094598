"""CPU oracle for the row-splitting solve phase -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.  The product package (paper_2603_28642_b200)
never imports it; its hot path fails loudly without the CUDA library.

This is a restatement of the reference package `rowsplit` (read-only at
/root/reference/pkg/src/rowsplit; cited as sc.py = sparse_core.py,
pc.py = precond.py, sv.py = solver.py).  The sparse kernels run in
oracle/rsref.c in the reference's exact floating-point order (bitwise
equal, pinned by tests/test_oracle_pin.py against fixtures generated from
the reference itself); the host loops below follow the reference line by
line.  Every ``a @ b`` / ``np.linalg.norm`` of the reference goes through
``dot`` / ``norm`` below, which restate OpenBLAS ddot in the association
order the reference host uses single-threaded (rsref.c rso_blas_dot), so
the oracle is bit-identical to the reference with OPENBLAS_NUM_THREADS=1 on
that host and host-independent everywhere else.

Inputs are duck-typed: any object with nrows/ncols/col_ptr/row_idx/values
is a CSC matrix, so reference objects and the product package's objects
both work.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liboracle_rsref.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            build()
        L = ctypes.CDLL(_SO)
        i64, f64 = ctypes.c_int64, ctypes.c_double
        L.rso_matvec.argtypes = [i64, i64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.rso_matvec_transpose.argtypes = [i64, i64, _i64p, _i64p, _f64p, _f64p, _f64p, _f64p]
        L.rso_lower_solve.argtypes = [i64, _i64p, _i64p, _f64p, _f64p, _f64p, ctypes.c_int]
        L.rso_lower_solve.restype = i64
        L.rso_upper_solve.argtypes = [i64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.rso_upper_solve.restype = i64
        L.rso_lower_solve_transpose.argtypes = [i64, _i64p, _i64p, _f64p, _f64p, _f64p, ctypes.c_int]
        L.rso_lower_solve_transpose.restype = i64
        L.rso_upper_solve_transpose.argtypes = [i64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.rso_upper_solve_transpose.restype = i64
        L.rso_cholesky_factorize.argtypes = [i64, _f64p]
        L.rso_cholesky_factorize.restype = i64
        L.rso_cholesky_solve.argtypes = [i64, _f64p, _f64p, _f64p]
        L.rso_pairwise_sum.argtypes = [_f64p, i64]
        L.rso_pairwise_sum.restype = f64
        L.rso_blas_dot.argtypes = [i64, _f64p, _f64p]
        L.rso_blas_dot.restype = f64
        # rsfast.c (threaded evaluation, same bits)
        L.rsf_csr.argtypes = [i64, i64, _i64p, _i64p, _f64p, _i64p, _i64p, _f64p]
        L.rsf_matvec_csr.argtypes = [i64, _i64p, _i64p, _f64p, _f64p, _f64p]
        L.rsf_matvec_t.argtypes = [i64, _i64p, _i64p, _f64p, _f64p, _f64p, i64]
        L.rsf_levels.argtypes = [i64, _i64p, _i64p, ctypes.c_int, _i64p, _i64p]
        L.rsf_levels.restype = i64
        for nm in ("rsf_lower_unit", "rsf_upper", "rsf_lower_t_unit"):
            getattr(L, nm).argtypes = [i64, _i64p, _i64p, _f64p, _f64p, _f64p, i64, _i64p, _i64p]
        L.rsf_dot.argtypes = [i64, _f64p, _f64p, ctypes.c_int]
        L.rsf_dot.restype = f64
        L.rsf_axpy.argtypes = [i64, _f64p, f64, _f64p, ctypes.c_int]
        L.rsf_xpby.argtypes = [i64, _f64p, _f64p, f64, _f64p]
        L.rsf_gather.argtypes = [i64, _f64p, _f64p, _i64p]
        L.rsf_sub.argtypes = [i64, _f64p, _f64p, _f64p]
        L.rsf_add.argtypes = [i64, _f64p, _f64p, _f64p]
        L.rsf_copy.argtypes = [i64, _f64p, _f64p]
        L.rsf_scale_div.argtypes = [i64, _f64p, _f64p, f64]
        L.rsf_max_threads.restype = ctypes.c_int
        L.rsf_set_threads.argtypes = [ctypes.c_int]
        # ilupref.c
        L.orc_ilup_factorize.argtypes = [i64, i64, _i64p, _i64p, _f64p, i64, f64, f64, f64,
                                         ctypes.POINTER(ctypes.c_void_p), _i64p]
        L.orc_ilup_sizes.argtypes = [ctypes.c_void_p, _i64p, _i64p, _i64p, _i64p]
        L.orc_ilup_copy.argtypes = [ctypes.c_void_p] + [_i64p, _i64p, _i64p, _i64p, _f64p, _i64p, _i64p,
                                                        _f64p, _i64p, _i64p, _f64p]
        L.orc_ilup_free.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


def _p64(a):
    return a.ctypes.data_as(_i64p)


def _pf(a):
    return a.ctypes.data_as(_f64p)


def _csc(A):
    cp = np.ascontiguousarray(A.col_ptr, dtype=np.int64)
    ri = np.ascontiguousarray(A.row_idx, dtype=np.int64)
    va = np.ascontiguousarray(A.values, dtype=np.float64)
    return int(A.nrows), int(A.ncols), cp, ri, va


def _vec(v, n):
    v = np.ascontiguousarray(v, dtype=np.float64)
    if v.shape != (n,):
        raise ValueError(f"vector has shape {v.shape}, expected ({n},)")
    return v


# ---------------------------------------------------------------------------
# threaded evaluation (rsfast.c): the same bits on all host cores
# ---------------------------------------------------------------------------

_cpu_threads = int(os.environ.get("RSB_ORACLE_THREADS", "1") or 1)


def set_cpu_threads(t: int) -> int:
    """Host threads the oracle kernels use (1 = the sequential restatement).
    Results are bit-identical either way; returns the previous value."""
    global _cpu_threads
    prev, _cpu_threads = _cpu_threads, max(1, int(t))
    lib().rsf_set_threads(_cpu_threads)
    return prev


def available_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        return os.cpu_count() or 1


class _Prep:
    """Per-matrix data of the threaded kernels: the CSC arrays, a CSR copy
    and the dependency levels of each solve kind, built on first use."""

    def __init__(self, M):
        self.M = M  # keeps id(M) unique while cached
        self.m, self.n, self.cp, self.ri, self.va = _csc(M)
        self.maxcol = int(np.diff(self.cp).max()) if self.n else 0
        self._csr = None
        self._lev = {}
        self._upper_ok = None

    def csr(self):
        if self._csr is None:
            nnz = int(self.cp[-1])
            rp, ci, rv = np.empty(self.m + 1, dtype=np.int64), np.empty(nnz, dtype=np.int64), np.empty(nnz)
            lib().rsf_csr(self.m, self.n, _p64(self.cp), _p64(self.ri), _pf(self.va), _p64(rp), _p64(ci), _pf(rv))
            self._csr = (rp, ci, rv)
        return self._csr

    def upper_ok(self):
        """every column's last stored entry is a nonzero diagonal (else the
        sequential path raises LinAlgError as the reference does)"""
        if self._upper_ok is None:
            cp, ri, va = self.cp, self.ri, self.va
            last = cp[1:] - 1
            ok = self.m == self.n and bool(np.all(cp[1:] > cp[:-1]))
            if ok:
                ok = bool(np.all(ri[last] == np.arange(self.n))) and bool(np.all(va[last] != 0.0))
            self._upper_ok = ok
        return self._upper_ok

    def levels(self, kind):
        if kind not in self._lev:
            if kind == 2:
                ptr, idx = self.cp, self.ri
            else:
                ptr, idx = self.csr()[0], self.csr()[1]
            order = np.empty(self.n, dtype=np.int64)
            lp = np.empty(self.n + 1, dtype=np.int64)
            nl = lib().rsf_levels(self.n, _p64(ptr), _p64(idx), kind, _p64(order), _p64(lp))
            self._lev[kind] = (int(nl), order, lp)
        return self._lev[kind]

    def solve(self, kind, b):
        """kind 0: unit lower (strict lower L), 1: upper, 2: unit lower transpose"""
        b = _vec(b, self.n)
        x = np.empty(self.n)
        nl, order, lp = self.levels(kind)
        if kind == 2:
            lib().rsf_lower_t_unit(self.n, _p64(self.cp), _p64(self.ri), _pf(self.va), _pf(b), _pf(x), nl,
                                   _p64(order), _p64(lp))
        else:
            rp, ci, rv = self.csr()
            fn = lib().rsf_lower_unit if kind == 0 else lib().rsf_upper
            fn(self.n, _p64(rp), _p64(ci), _pf(rv), _pf(b), _pf(x), nl, _p64(order), _p64(lp))
        return x


_preps: dict = {}


def _prep(M):
    P = _preps.get(id(M))
    if P is None or P.M is not M:
        P = _preps[id(M)] = _Prep(M)
    return P


def clear_prep_cache():
    _preps.clear()


# elementwise steps of the loops below, one IEEE operation per element as
# numpy performs them; threaded when _cpu_threads > 1
def _axpy(y, a, x, sign):
    """y += a*x (sign +1) / y -= a*x (sign -1), in place"""
    if _cpu_threads > 1:
        lib().rsf_axpy(len(y), _pf(y), float(a), _pf(x), sign)
    elif sign > 0:
        y += a * x
    else:
        y -= a * x


def _xpby(h, beta, p):
    """h + beta*p (new array)"""
    if _cpu_threads > 1:
        out = np.empty(len(h))
        lib().rsf_xpby(len(h), _pf(out), _pf(h), float(beta), _pf(p))
        return out
    return h + beta * p


def _add(a, b):
    if _cpu_threads > 1:
        a, b = np.ascontiguousarray(a, dtype=np.float64), np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty(len(a))
        lib().rsf_add(len(a), _pf(out), _pf(a), _pf(b))
        return out
    return a + b


def _sub(a, b):
    if _cpu_threads > 1:
        a, b = np.ascontiguousarray(a, dtype=np.float64), np.ascontiguousarray(b, dtype=np.float64)
        out = np.empty(len(a))
        lib().rsf_sub(len(a), _pf(out), _pf(a), _pf(b))
        return out
    return a - b


def _copy(a):
    if _cpu_threads > 1:
        a = np.ascontiguousarray(a, dtype=np.float64)
        out = np.empty(len(a))
        lib().rsf_copy(len(a), _pf(out), _pf(a))
        return out
    return np.array(a, dtype=np.float64, copy=True)


def _gather(r, perm):
    if _cpu_threads > 1:
        out = np.empty(len(perm))
        lib().rsf_gather(len(perm), _pf(out), _pf(r), _p64(perm))
        return out
    return r[perm]


# ---------------------------------------------------------------------------
# kernels (sc.py)
# ---------------------------------------------------------------------------


def matvec(A, x):
    """sc.py:212-221."""
    m, n, cp, ri, va = _csc(A)
    x = _vec(x, n)
    y = np.empty(m)
    if _cpu_threads > 1:
        P = _prep(A)
        rp, ci, rv = P.csr()
        lib().rsf_matvec_csr(m, _p64(rp), _p64(ci), _pf(rv), _pf(x), _pf(y))
        return y
    lib().rso_matvec(m, n, _p64(cp), _p64(ri), _pf(va), _pf(x), _pf(y))
    return y


def matvec_transpose(A, y):
    """sc.py:224-235."""
    m, n, cp, ri, va = _csc(A)
    y = _vec(y, m)
    z = np.empty(n)
    if _cpu_threads > 1:
        P = _prep(A)
        lib().rsf_matvec_t(n, _p64(P.cp), _p64(P.ri), _pf(P.va), _pf(y), _pf(z), P.maxcol)
        return z
    scratch = np.empty(max(1, int(np.diff(cp).max()) if n else 1))
    lib().rso_matvec_transpose(m, n, _p64(cp), _p64(ri), _pf(va), _pf(y), _pf(z), _pf(scratch))
    return z


def _tri(fn, T, b, *extra):
    m, n, cp, ri, va = _csc(T)
    if m != n:
        raise ValueError("triangular solve needs a square matrix")
    b = _vec(b, n)
    x = np.empty(n)
    rc = fn(n, _p64(cp), _p64(ri), _pf(va), _pf(b), _pf(x), *extra)
    if rc < 0:
        raise np.linalg.LinAlgError(f"missing or zero diagonal in column {-rc - 1}")
    return x


def sparse_lower_solve(L, b, unit_diag=False):
    """sc.py:243-263."""
    if _cpu_threads > 1 and unit_diag:
        return _prep(L).solve(0, b)
    return _tri(lib().rso_lower_solve, L, b, int(bool(unit_diag)))


def sparse_upper_solve(U, b):
    """sc.py:266-279."""
    if _cpu_threads > 1 and _prep(U).upper_ok():
        return _prep(U).solve(1, b)
    return _tri(lib().rso_upper_solve, U, b)


def sparse_lower_solve_transpose(L, b, unit_diag=False):
    """sc.py:282-298."""
    if _cpu_threads > 1 and unit_diag and _prep(L).maxcol <= 256:
        return _prep(L).solve(2, b)
    return _tri(lib().rso_lower_solve_transpose, L, b, int(bool(unit_diag)))


def sparse_upper_solve_transpose(U, b):
    """sc.py:301-313."""
    return _tri(lib().rso_upper_solve_transpose, U, b)


def dense_cholesky_factorize(S):
    """sc.py:585-604; S is an (s, s) array; returns the lower factor (Fortran order)."""
    g = np.array(S, dtype=np.float64, order="F", copy=True)
    s = g.shape[0]
    rc = lib().rso_cholesky_factorize(s, _pf(g))
    if rc < 0:
        raise np.linalg.LinAlgError(f"matrix is not positive definite (pivot {-rc - 1})")
    return g


def dense_cholesky_solve(g, b):
    """sc.py:607-622; g is the lower factor as an (s, s) array."""
    g = np.asfortranarray(g, dtype=np.float64)
    s = g.shape[0]
    b = _vec(b, s)
    x = np.empty(s)
    lib().rso_cholesky_solve(s, _pf(g), _pf(b), _pf(x))
    return x


_blas_threads = int(os.environ.get("RSB_BLAS_THREADS", "1") or 1)


def set_blas_threads(t: int) -> int:
    """OpenBLAS thread count T the reference ran with (OPENBLAS_NUM_THREADS=T
    on a host with >= T cores); returns the previous value."""
    global _blas_threads
    if not 1 <= int(t) <= 64:
        raise ValueError("blas threads must be in 1..64")
    prev, _blas_threads = _blas_threads, int(t)
    return prev


def blas_chunks(n: int, t: int) -> list[int]:
    """OpenBLAS's split of an n-long ddot over t threads
    (driver/others/blas_l1_thread.c): n <= 10000 runs on one thread,
    otherwise widths ceil(rest / threads left)."""
    if t <= 1 or n <= 10000:
        return [n]
    out, rest = [], n
    for i in range(t):
        w = -(-rest // (t - i))
        out.append(w)
        rest -= w
    return out


def dot(a, b):
    """`a @ b` for 1-D float64 as the reference host's OpenBLAS computes it
    (rsref.c rso_blas_dot per thread; with T threads the chunk results are
    summed in thread order from 0.0, interface/dot.c)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    if a.shape != b.shape:
        raise ValueError("dot: shape mismatch")
    widths = blas_chunks(len(a), _blas_threads)
    if len(widths) == 1:
        return lib().rso_blas_dot(len(a), _pf(a), _pf(b))
    if _cpu_threads > 1:
        return lib().rsf_dot(len(a), _pf(a), _pf(b), _blas_threads)
    total, lo = 0.0, 0
    for w in widths:
        total = total + lib().rso_blas_dot(w, _pf(a[lo:lo + w]), _pf(b[lo:lo + w]))
        lo += w
    return total


def norm(a):
    """np.linalg.norm of a 1-D float64 vector: sqrt(a.dot(a))."""
    return float(np.sqrt(dot(a, a)))


def pairwise_sum(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().rso_pairwise_sum(_pf(a), len(a))


def power_method_norm2(A, iters=100, seed=0):
    """sc.py:428-454."""
    if iters < 1:
        raise ValueError("iters must be >= 1")
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(int(A.ncols))
    nv = norm(v)
    if nv == 0.0 or int(A.col_ptr[-1]) == 0:
        return 0.0
    v /= nv
    est = 0.0
    for _ in range(iters):
        w = matvec(A, v)
        est = norm(w)
        if est == 0.0:
            return 0.0
        t = matvec_transpose(A, w)
        nt = norm(t)
        if nt == 0.0:
            return est
        if _cpu_threads > 1:
            v = np.empty(len(t))
            lib().rsf_scale_div(len(t), _pf(v), _pf(t), float(nt))
        else:
            v = t / nt
    return float(est)


# ---------------------------------------------------------------------------
# preconditioner application (pc.py)
# ---------------------------------------------------------------------------


class OraclePreconditioner:
    """Applied row-splitting preconditioner, pc.py:106-186.

    factors: object with L1, L2, U (CSC), row_perm.perm, nmod.
    s_mode: "dense" | "cg" | "identity"; y_mode: "explicit" | "implicit".
    Y (CSC, explicit mode) and S_factor (s x s lower array, dense mode)
    come from the caller (built by the reference or by the product setup).
    """

    def __init__(self, factors, s_mode, y_mode, cg_iters=2, Y=None, S_factor=None, psize=0):
        self.factors = factors
        self.s_mode = s_mode
        self.y_mode = y_mode
        self.cg_iters = cg_iters
        self.Y = Y
        self.S_factor = None if S_factor is None else np.asfortranarray(S_factor)
        self.psize = psize

    @classmethod
    def from_reference(cls, pre):
        """Wrap a reference RowSplitPreconditioner (or a product one)."""
        S = getattr(pre, "S_factor", None)
        S = None if S is None else getattr(S, "a", S)
        sm = getattr(pre.s_mode, "value", pre.s_mode)
        ym = getattr(pre.y_mode, "value", pre.y_mode)
        return cls(pre.factors, sm, ym, pre.cg_iters, pre.Y, S, pre.psize)

    @property
    def n(self):
        return int(self.factors.U.ncols)

    @property
    def split_rows(self):
        return int(self.factors.L2.nrows)

    def y_apply(self, r1):
        """pc.py:135-139."""
        if self.y_mode == "explicit":
            return matvec(self.Y, r1)
        f = self.factors
        return matvec(f.L2, sparse_lower_solve(f.L1, r1, unit_diag=True))

    def y_apply_transpose(self, w):
        """pc.py:141-147."""
        if self.y_mode == "explicit":
            return matvec_transpose(self.Y, w)
        f = self.factors
        return sparse_lower_solve_transpose(f.L1, matvec_transpose(f.L2, w), unit_diag=True)

    def s_matvec_implicit(self, v):
        """pc.py:149-154."""
        f = self.factors
        v = np.asarray(v, dtype=np.float64)
        t = matvec_transpose(f.L2, v)
        t = sparse_lower_solve_transpose(f.L1, t, unit_diag=True)
        t = sparse_lower_solve(f.L1, t, unit_diag=True)
        return _add(v, matvec(f.L2, t))

    def _solve_s(self, u):
        """pc.py:158-163."""
        if self.s_mode == "dense":
            return dense_cholesky_solve(self.S_factor, u)
        if self.s_mode == "identity":
            return _copy(u)
        return cg_fixed_steps(self.s_matvec_implicit, u, self.cg_iters)

    def apply(self, r1, r2):
        """pc.py:167-186."""
        r1 = np.asarray(r1, dtype=np.float64)
        r2 = np.asarray(r2, dtype=np.float64)
        if r1.shape != (self.n,) or r2.shape != (self.split_rows,):
            raise ValueError("residual component lengths do not match the split")
        if self.split_rows:
            u = _sub(r2, self.y_apply(r1))
            w = self._solve_s(u)
            y = _add(r1, self.y_apply_transpose(w))
        else:
            y = r1
        v = sparse_lower_solve(self.factors.L1, y, unit_diag=True)
        return sparse_upper_solve(self.factors.U, v)


def cg_fixed_steps(op, u, iters):
    """pc.py:284-310."""
    w = np.zeros(len(u))
    r = _copy(u)
    rho = dot(r, r)
    if rho == 0.0:
        return w
    p = _copy(r)
    for _ in range(iters):
        q = op(p)
        pq = dot(p, q)
        if pq <= 0.0:
            break
        alpha = rho / pq
        _axpy(w, alpha, p, +1)
        _axpy(r, alpha, q, -1)
        rho_new = dot(r, r)
        if rho_new == 0.0:
            break
        p = _xpby(r, rho_new / rho, p)
        rho = rho_new
    return w


# ---------------------------------------------------------------------------
# solver (sv.py)
# ---------------------------------------------------------------------------


def stopping_ratio(estim, norm_A, x_norm, b_norm, raw=False):
    """sv.py:104-117."""
    denom = norm_A * x_norm + b_norm
    if denom <= 0.0:
        raise ValueError("zero denominator in stopping ratio")
    if estim < 0.0:
        estim = 0.0
    num = estim if raw else np.sqrt(estim)
    return float(num / denom)


def pcgls(A, b, pre, norm_A, delta=1e-10, max_iters=2000, d=5, ratio_raw=False,
          iterate_hook=None):
    """sv.py:120-268.  Returns (x, report dict with SolveReport.to_dict keys)."""
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (int(A.nrows),):
        raise ValueError("right-hand side length mismatch")
    n = int(A.ncols)
    b_norm = float(norm(b))
    if pre is not None:
        perm = np.ascontiguousarray(pre.factors.row_perm.perm, dtype=np.int64)

        def precondition(r):
            rp = _gather(r, perm)
            return pre.apply(rp[:n], rp[n:])

        psize, nmod = pre.psize, pre.factors.nmod
    else:

        def precondition(r):
            return matvec_transpose(A, r)

        psize, nmod = 0, 0

    def report(its, converged, breakdown, history, res, grad):
        return {
            "its": its, "converged": converged, "breakdown": breakdown,
            "ratio_pt": history[-1] if history else float("inf"),
            "ratio_pt_history": list(history), "psize": psize, "nmod": nmod,
            "residual_norm": res, "gradient_norm": grad,
        }

    x = np.zeros(n)
    r = _copy(b)
    z = matvec_transpose(A, r)
    alphas, sigmas, x_norms, history = [], [], [0.0], []
    converged = False
    its_certified = 0
    iters_run = 0
    if float(dot(z, z)) == 0.0:
        return x, report(0, True, False, [0.0], b_norm, 0.0)

    h = precondition(r)
    rho = float(dot(z, h))
    p = _copy(h)
    stopped_early = False
    for it in range(max_iters):
        sigma = rho if rho > 0.0 else float(dot(z, p))
        if sigma == 0.0:
            p = _copy(z)
            sigma = float(dot(z, z))
            rho = sigma
        q = matvec(A, p)
        qq = float(dot(q, q))
        if qq <= 0.0 or sigma == 0.0:
            stopped_early = True
            break
        alpha = sigma / qq
        _axpy(x, alpha, p, +1)
        _axpy(r, alpha, q, -1)
        alphas.append(alpha)
        sigmas.append(sigma)
        x_norms.append(float(norm(x)))
        iters_run = it + 1
        if iterate_hook is not None:
            iterate_hook(iters_run, x.copy())
        i = iters_run - d
        if i >= 0:
            estim = float(sum(a * s for a, s in zip(alphas[i:], sigmas[i:])))
            ratio = stopping_ratio(estim, norm_A, x_norms[i], b_norm, raw=ratio_raw)
            history.append(ratio)
            if ratio <= delta:
                converged = True
                its_certified = i
                break
        z = matvec_transpose(A, r)
        if float(dot(z, z)) == 0.0:
            stopped_early = True
            break
        h = precondition(r)
        rho_new = float(dot(z, h))
        p = _xpby(h, rho_new / rho, p) if rho != 0.0 else _copy(h)
        rho = rho_new

    if stopped_early and not converged:
        for i in range(max(0, iters_run - d + 1), iters_run + 1):
            estim = float(sum(a * s for a, s in zip(alphas[i:], sigmas[i:])))
            ratio = stopping_ratio(estim, norm_A, x_norms[i], b_norm, raw=ratio_raw)
            history.append(ratio)
            if ratio <= delta:
                converged = True
                its_certified = i
                break

    its = its_certified if converged else iters_run
    fr = _sub(b, matvec(A, x))
    return x, report(its, converged, stopped_early and not converged, history,
                     float(norm(fr)), float(norm(matvec_transpose(A, fr))))


# ---------------------------------------------------------------------------
# host setup (reference arm of bench.py: sets the configs up with no product
# code) -- column_scale sc.py:405-425, ilup_factorize il.py:211-368
# ---------------------------------------------------------------------------


class Csc:
    """Minimal CscMatrix (sc.py:27-131 fields): int64 col_ptr/row_idx, f64 values."""

    def __init__(self, nrows, ncols, col_ptr, row_idx, values):
        self.nrows, self.ncols = int(nrows), int(ncols)
        self.col_ptr, self.row_idx, self.values = col_ptr, row_idx, values

    @property
    def nnz(self):
        return int(self.col_ptr[-1])

    def column_counts(self):
        return np.diff(self.col_ptr)


class _Perm:
    def __init__(self, perm):
        self.perm = perm


class Factors:
    """IlupFactors fields (il.py:53-77)."""

    def __init__(self, perm, L1, L2, U, nmod, row_counts):
        self.row_perm, self.L1, self.L2, self.U = _Perm(perm), L1, L2, U
        self.nmod, self.row_counts_final = nmod, row_counts


def column_scale(A):
    """sc.py:405-425 with numpy's own reduceat / sqrt / divide (the same
    calls the reference makes).  Returns (scaled Csc, norms)."""
    counts = np.diff(A.col_ptr)
    empty = np.flatnonzero(counts == 0)
    if len(empty):
        raise ValueError(f"cannot scale zero column {empty[0]}")
    sq = np.zeros(A.ncols)
    sq[:] = np.add.reduceat(A.values * A.values, A.col_ptr[:-1])
    norms = np.sqrt(sq)
    S = Csc(A.nrows, A.ncols, A.col_ptr.copy(), A.row_idx.copy(), A.values / np.repeat(norms, counts))
    return S, norms


def ilup_factorize(A, p=10, tau=0.0, mu=0.1, small=1e-10):
    """il.py:211-368 (oracle/ilupref.c).  Returns Factors."""
    m, n, cp, ri, va = _csc(A)
    h = ctypes.c_void_p()
    err = ctypes.c_int64(-1)
    rc = lib().orc_ilup_factorize(m, n, _p64(cp), _p64(ri), _pf(va), int(p), float(tau), float(mu),
                                  float(small), ctypes.byref(h), ctypes.byref(err))
    if rc == 1:
        raise ValueError("invalid ILUP input or parameters")
    if rc == 2:
        raise np.linalg.LinAlgError(f"non-finite value in column {err.value} of the factorization")
    if rc != 0:
        raise MemoryError("oracle ILUP: out of memory")
    try:
        n1, n2, nu, nm = (ctypes.c_int64() for _ in range(4))
        lib().orc_ilup_sizes(h, ctypes.byref(n1), ctypes.byref(n2), ctypes.byref(nu), ctypes.byref(nm))
        perm, rcnt = np.empty(m, dtype=np.int64), np.empty(m, dtype=np.int64)
        l1p, l2p, up = (np.empty(n + 1, dtype=np.int64) for _ in range(3))
        l1i, l1v = np.empty(n1.value, dtype=np.int64), np.empty(n1.value)
        l2i, l2v = np.empty(n2.value, dtype=np.int64), np.empty(n2.value)
        ui, uv = np.empty(nu.value, dtype=np.int64), np.empty(nu.value)
        lib().orc_ilup_copy(h, _p64(perm), _p64(rcnt), _p64(l1p), _p64(l1i), _pf(l1v), _p64(l2p), _p64(l2i),
                            _pf(l2v), _p64(up), _p64(ui), _pf(uv))
    finally:
        lib().orc_ilup_free(h)
    return Factors(perm, Csc(n, n, l1p, l1i, l1v), Csc(m - n, n, l2p, l2i, l2v), Csc(n, n, up, ui, uv),
                   int(nm.value), rcnt)
