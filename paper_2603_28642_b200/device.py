"""Device-side handles: contexts, uploaded matrices, preconditioners, solvers.

Thin owners of the C-ABI handles (include/rowsplit_b200.h).  The public
reference-shaped API (sparse.py, precond.py, solver.py) builds on these;
bench.py uses them directly for device-resident timing.
"""

from __future__ import annotations

import atexit
import collections
import ctypes
import os
import threading

import numpy as np

from . import _lib as L

_ctx_lock = threading.Lock()
_contexts: dict[tuple, "Context"] = {}
_exiting = False


@atexit.register
def _at_exit():
    # Interpreter teardown finalizes objects in no particular order; device
    # handles are left to process exit (the driver reclaims the context)
    # instead of being destroyed against an already-destroyed rsb_ctx.
    global _exiting
    _exiting = True


def _alive(obj, attr="h"):
    return not _exiting and getattr(obj, attr, None)


def device_count() -> int:
    c = ctypes.c_int(0)
    L.check(L.lib().rsb_device_count(ctypes.byref(c)))
    return c.value


def default_device() -> int:
    env = os.environ.get("RSB_DEVICE")
    if env is not None:
        return int(env)
    return int(os.environ.get("LOCAL_RANK", "0"))


def blas_threads() -> int:
    """OpenBLAS thread count whose ddot association the exact dot order
    reproduces (RSB_BLAS_THREADS, default 1: the reference run with
    OPENBLAS_NUM_THREADS=1).  The reference's numpy splits a dot longer than
    10000 over min(OPENBLAS_NUM_THREADS, cores) threads, at most 64."""
    t = int(os.environ.get("RSB_BLAS_THREADS", "1") or 1)
    if not 1 <= t <= 64:
        raise ValueError("RSB_BLAS_THREADS must be in 1..64")
    return t


def dot_flags() -> int:
    if os.environ.get("RSB_DOT_ORDER", "exact") == "tree":
        return L.RSB_DOT_TREE
    t = blas_threads()
    return L.RSB_DOT_EXACT | ((t << 8) if t > 1 else 0)


class Context:
    """One CUDA stream on one device (rsb_ctx)."""

    def __init__(self, device: int | None = None, flags: int | None = None):
        self.device = default_device() if device is None else device
        self.flags = dot_flags() if flags is None else flags
        h = ctypes.c_void_p()
        L.check(L.lib().rsb_ctx_create(self.device, self.flags, ctypes.byref(h)))
        self.h = h

    def sync(self):
        L.check(L.lib().rsb_ctx_sync(self.h))

    def kernel_launches(self, reset=False) -> int:
        c = ctypes.c_int64()
        L.check(L.lib().rsb_ctx_kernel_launches(self.h, ctypes.byref(c), int(reset)))
        return c.value

    def mem_bytes(self) -> int:
        c = ctypes.c_int64()
        L.check(L.lib().rsb_ctx_mem_bytes(self.h, ctypes.byref(c)))
        return c.value

    def mark(self, slot: int):
        L.check(L.lib().rsb_event_mark(self.h, slot))

    def elapsed_ms(self, s0: int, s1: int) -> float:
        ms = ctypes.c_float()
        L.check(L.lib().rsb_event_elapsed(self.h, s0, s1, ctypes.byref(ms)))
        return float(ms.value)

    def __del__(self):
        try:
            if _alive(self):
                L.lib().rsb_ctx_destroy(self.h)
                self.h = None
        except Exception:
            pass


def get_context(device: int | None = None) -> Context:
    dev = default_device() if device is None else device
    flags = dot_flags()
    with _ctx_lock:
        ctx = _contexts.get((dev, flags))
        if ctx is None:
            ctx = Context(dev, flags)
            _contexts[(dev, flags)] = ctx
        return ctx


class DeviceBuffer:
    """Raw device allocation (float64 vector) owned by a context."""

    def __init__(self, ctx: Context, n: int):
        self.ctx, self.n = ctx, int(n)
        p = ctypes.c_void_p()
        L.check(L.lib().rsb_device_alloc(ctx.h, max(8, 8 * self.n), ctypes.byref(p)))
        self.ptr = p

    def upload(self, a):
        a = L.f64c(a)
        assert a.size == self.n
        L.check(L.lib().rsb_memcpy(self.ctx.h, self.ptr, L.ptr(a), 8 * self.n, 0))
        self.ctx.sync()

    def download(self):
        out = np.empty(self.n)
        L.check(L.lib().rsb_memcpy(self.ctx.h, L.ptr(out), self.ptr, 8 * self.n, 1))
        self.ctx.sync()
        return out

    def __del__(self):
        try:
            if _alive(self, "ptr"):
                L.lib().rsb_device_free(self.ctx.h, self.ptr)
                self.ptr = None
        except Exception:
            pass


class PinnedBuffer:
    """Page-locked host float64 vector (for timed host<->device copies)."""

    def __init__(self, n: int):
        self.n = int(n)
        p = ctypes.c_void_p()
        L.check(L.lib().rsb_host_alloc(max(8, 8 * self.n), ctypes.byref(p)))
        self.ptr = p
        self.array = np.ctypeslib.as_array((ctypes.c_double * max(1, self.n)).from_address(p.value))[: self.n]

    def __del__(self):
        try:
            if _alive(self, "ptr"):
                self.array = None
                L.lib().rsb_host_free(self.ptr)
                self.ptr = None
        except Exception:
            pass


class DeviceMatrix:
    """A CSC matrix uploaded as device CSR + CSC (rsb_mat)."""

    def __init__(self, A, ctx: Context | None = None):
        self.ctx = ctx or get_context()
        self.nrows, self.ncols = int(A.nrows), int(A.ncols)
        cp = L.i64c(A.col_ptr)
        ri = L.i64c(A.row_idx)
        va = L.f64c(A.values)
        if cp.shape != (self.ncols + 1,):
            raise ValueError("col_ptr has wrong length")
        if len(ri) != len(va) or cp[-1] != len(ri):
            raise ValueError("col_ptr endpoints inconsistent with storage")
        h = ctypes.c_void_p()
        L.check(L.lib().rsb_mat_create(self.ctx.h, self.nrows, self.ncols, L.ptr(cp), L.ptr(ri),
                                       L.ptr(va), ctypes.byref(h)))
        self.h = h
        self.nnz = int(cp[-1])

    def variant(self, kind: int) -> tuple[str, int]:
        """(kernel family, longest task of the lean kernel or 0) of a solve."""
        v, n = ctypes.c_int(), ctypes.c_int()
        L.check(L.lib().rsb_trsv_variant(self.h, kind, ctypes.byref(v), ctypes.byref(n)))
        return ("grid", "staged", "lean", "levels", "lsync", "levelsync", "natural")[v.value], n.value

    def levels(self, kind: int):
        nl, mw = ctypes.c_int64(), ctypes.c_int64()
        L.check(L.lib().rsb_trsv_levels(self.h, kind, ctypes.byref(nl), ctypes.byref(mw)))
        return nl.value, mw.value

    def __del__(self):
        try:
            if _alive(self):
                L.lib().rsb_mat_destroy(self.h)
                self.h = None
        except Exception:
            pass


# Uploaded matrices are cached per host object so repeated calls with the
# same matrix do not re-upload.  Keys are id()s; the cache holds the host
# object too, so an id cannot be recycled while its entry lives.
_MAT_CACHE_SIZE = 32
_mat_cache: "collections.OrderedDict[tuple, tuple]" = collections.OrderedDict()


def device_matrix(A, ctx: Context | None = None) -> DeviceMatrix:
    ctx = ctx or get_context()
    key = (id(A), id(ctx))
    hit = _mat_cache.get(key)
    if hit is not None and hit[0] is A:
        _mat_cache.move_to_end(key)
        return hit[1]
    dm = DeviceMatrix(A, ctx)
    _mat_cache[key] = (A, dm)
    while len(_mat_cache) > _MAT_CACHE_SIZE:
        _mat_cache.popitem(last=False)
    return dm


def clear_caches():
    _bsolver_cache.clear()
    _batch_cache.clear()
    _mat_cache.clear()
    _pre_cache.clear()
    _solver_cache.clear()


S_MODE_CODE = {"dense": L.S_DENSE, "cg": L.S_CG, "identity": L.S_IDENTITY}
Y_MODE_CODE = {"explicit": L.Y_EXPLICIT, "implicit": L.Y_IMPLICIT}


def _mode_value(m):
    return getattr(m, "value", m)


class DevicePreconditioner:
    """Device form of a RowSplitPreconditioner (rsb_pre)."""

    def __init__(self, pre, ctx: Context | None = None):
        self.ctx = ctx or get_context()
        f = pre.factors
        self.n = int(f.U.ncols)
        self.s = int(f.L2.nrows)
        self.m = self.n + self.s
        self.L1 = DeviceMatrix(f.L1, self.ctx)
        self.L2 = DeviceMatrix(f.L2, self.ctx)
        self.U = DeviceMatrix(f.U, self.ctx)
        sm = S_MODE_CODE[_mode_value(pre.s_mode)]
        ym = Y_MODE_CODE[_mode_value(pre.y_mode)]
        self.Y = DeviceMatrix(pre.Y, self.ctx) if (ym == L.Y_EXPLICIT and pre.Y is not None) else None
        S = None
        if sm == L.S_DENSE and self.s > 0:
            Sa = getattr(pre.S_factor, "a", pre.S_factor)
            S = np.asfortranarray(Sa, dtype=np.float64)
        perm = L.i64c(f.row_perm.perm)
        h = ctypes.c_void_p()
        L.check(L.lib().rsb_pre_create(
            self.ctx.h, self.m, self.n, L.ptr(perm), self.L1.h, self.L2.h, self.U.h,
            self.Y.h if self.Y is not None else None,
            L.ptr(S.ravel(order="F")) if S is not None else None, self.s,
            sm, ym, int(pre.cg_iters), ctypes.byref(h)))
        self.h = h

    def _call(self, fn, a, n_in, n_out):
        a = L.f64c(a)
        if a.shape != (n_in,):
            raise ValueError(f"vector has length {a.shape}, expected ({n_in},)")
        out = np.empty(n_out)
        L.check(fn(self.h, L.ptr(a), L.ptr(out), L.RSB_HOST))
        return out

    def apply(self, r1, r2):
        r1, r2 = L.f64c(r1), L.f64c(r2)
        if r1.shape != (self.n,) or r2.shape != (self.s,):
            raise ValueError("residual component lengths do not match the split")
        h = np.empty(self.n)
        L.check(L.lib().rsb_pre_apply(self.h, L.ptr(r1), L.ptr(r2), L.ptr(h), L.RSB_HOST))
        return h

    def y_apply(self, r1):
        return self._call(L.lib().rsb_pre_y_apply, r1, self.n, self.s)

    def y_apply_transpose(self, w):
        return self._call(L.lib().rsb_pre_y_apply_transpose, w, self.s, self.n)

    def s_matvec(self, v):
        return self._call(L.lib().rsb_pre_s_matvec, v, self.s, self.s)

    def __del__(self):
        try:
            if _alive(self):
                L.lib().rsb_pre_destroy(self.h)
                self.h = None
        except Exception:
            pass


_pre_cache: "collections.OrderedDict[tuple, tuple]" = collections.OrderedDict()


def device_preconditioner(pre, ctx: Context | None = None) -> DevicePreconditioner:
    ctx = ctx or get_context()
    key = (id(pre), id(ctx))
    hit = _pre_cache.get(key)
    if hit is not None and hit[0] is pre:
        _pre_cache.move_to_end(key)
        return hit[1]
    dp = DevicePreconditioner(pre, ctx)
    _pre_cache[key] = (pre, dp)
    while len(_pre_cache) > 8:
        _pre_cache.popitem(last=False)
    return dp


class DeviceSolver:
    """Workspace + captured iteration graph for pcgls on one (A, pre) pair."""

    def __init__(self, dA: DeviceMatrix, dpre: DevicePreconditioner | None, ctx: Context | None = None):
        self.dA, self.dpre = dA, dpre
        self.ctx = dA.ctx if ctx is None else ctx
        h = ctypes.c_void_p()
        L.check(L.lib().rsb_solver_create_on(self.ctx.h, dA.h, dpre.h if dpre is not None else None,
                                             ctypes.byref(h)))
        self.h = h

    @staticmethod
    def cfg_struct(norm_A, delta, max_iters, d, ratio_raw):
        return L.CglsCfgC(float(norm_A), float(delta), int(max_iters), int(d), int(bool(ratio_raw)))

    def start(self, b_ptr, where, cfg: "L.CglsCfgC") -> int:
        st = ctypes.c_int()
        L.check(L.lib().rsb_solver_start(self.h, b_ptr, where, ctypes.byref(cfg), ctypes.byref(st)))
        return st.value

    def iterate(self, k):
        it, st = ctypes.c_int64(), ctypes.c_int()
        L.check(L.lib().rsb_solver_iterate(self.h, int(k), ctypes.byref(it), ctypes.byref(st)))
        return it.value, st.value

    def get_x(self, out_ptr, where):
        L.check(L.lib().rsb_solver_get_x(self.h, out_ptr, where))

    def finish(self, max_hist: int):
        rep = L.ReportC()
        hist = np.empty(max(1, max_hist))
        L.check(L.lib().rsb_solver_finish(self.h, ctypes.byref(rep), L.ptr(hist), len(hist)))
        return rep, hist[: min(rep.history_len, len(hist))].copy()

    def __del__(self):
        try:
            if _alive(self):
                L.lib().rsb_solver_destroy(self.h)
                self.h = None
        except Exception:
            pass


_solver_cache: "collections.OrderedDict[tuple, DeviceSolver]" = collections.OrderedDict()


def device_solver(dA: DeviceMatrix, dpre: DevicePreconditioner | None) -> DeviceSolver:
    key = (id(dA), id(dpre))
    s = _solver_cache.get(key)
    if s is not None and s.dA is dA and s.dpre is dpre:
        _solver_cache.move_to_end(key)
        return s
    s = DeviceSolver(dA, dpre)
    _solver_cache[key] = s
    while len(_solver_cache) > 8:
        _solver_cache.popitem(last=False)
    return s


_stream_pool: dict[tuple, list[Context]] = {}


def stream_contexts(k: int, device: int | None = None) -> list[Context]:
    """k distinct contexts (streams) on one device for concurrent solves; the
    first is the device's default context."""
    dev = default_device() if device is None else device
    flags = dot_flags()
    with _ctx_lock:
        pool = _stream_pool.setdefault((dev, flags), [])
    first = get_context(dev)
    with _ctx_lock:
        while len(pool) < k - 1:
            pool.append(Context(dev, flags))
        return [first] + pool[: k - 1]


_batch_cache: "collections.OrderedDict[tuple, list[DeviceSolver]]" = collections.OrderedDict()


def device_solvers(dA: DeviceMatrix, dpre: DevicePreconditioner | None, k: int) -> list[DeviceSolver]:
    """k solvers sharing dA and dpre, one per stream."""
    key = (id(dA), id(dpre), k)
    s = _batch_cache.get(key)
    if s is not None and s[0].dA is dA and s[0].dpre is dpre:
        _batch_cache.move_to_end(key)
        return s
    ctxs = stream_contexts(k, dA.ctx.device)
    s = [device_solver(dA, dpre)] + [DeviceSolver(dA, dpre, c) for c in ctxs[1:]]
    _batch_cache[key] = s
    while len(_batch_cache) > 4:
        _batch_cache.popitem(last=False)
    return s


BATCH = 8  # right-hand sides per batched solver (csrc/bsolver.cu kBatch)


class DeviceBatchSolver:
    """Up to BATCH pcgls solves advanced together (rsb_bsolver): matrix and
    factor entries are read once for all of them."""

    def __init__(self, dA: DeviceMatrix, dpre: DevicePreconditioner | None):
        self.dA, self.dpre = dA, dpre
        self.ctx = dA.ctx
        h = ctypes.c_void_p()
        L.check(L.lib().rsb_bsolver_create(dA.h, dpre.h if dpre is not None else None, ctypes.byref(h)))
        self.h = h

    def start(self, B, cfg: "L.CglsCfgC", where=L.RSB_HOST):
        k = B.shape[0] if where == L.RSB_HOST else B[1]
        st = (ctypes.c_int * BATCH)()
        ptr = L.ptr(B) if where == L.RSB_HOST else B[0]
        L.check(L.lib().rsb_bsolver_start(self.h, int(k), ptr, where, ctypes.byref(cfg), st))
        return list(st)[:k]

    def iterate(self, k):
        done = ctypes.c_int()
        L.check(L.lib().rsb_bsolver_iterate(self.h, int(k), ctypes.byref(done)))
        return bool(done.value)

    def finish(self, k, n, cap):
        X = np.empty((k, n))
        reps = (L.ReportC * k)()
        hist = np.empty((k, max(1, cap)))
        L.check(L.lib().rsb_bsolver_finish(self.h, L.ptr(X), L.RSB_HOST, reps, L.ptr(hist), hist.shape[1]))
        return X, reps, hist

    def __del__(self):
        try:
            if _alive(self):
                L.lib().rsb_bsolver_destroy(self.h)
                self.h = None
        except Exception:
            pass


_bsolver_cache: "collections.OrderedDict[tuple, object]" = collections.OrderedDict()


def device_batch_solver(dA: DeviceMatrix, dpre: DevicePreconditioner | None):
    """The cached batched solver of (dA, dpre), or None when the problem
    does not fit the batched kernels (explicit Y / dense S, narrow DAGs)."""
    key = (id(dA), id(dpre))
    hit = _bsolver_cache.get(key)
    if hit is not None and hit[0] is dA and hit[1] is dpre:
        _bsolver_cache.move_to_end(key)
        return hit[2]
    try:
        s = DeviceBatchSolver(dA, dpre)
    except ValueError:
        s = None
    _bsolver_cache[key] = (dA, dpre, s)
    while len(_bsolver_cache) > 2:
        _bsolver_cache.popitem(last=False)
    return s
