"""Preconditioned CGLS with the reference's API; the iteration runs on the B200.

Mirrors pkg/src/rowsplit/solver.py (sv.py): CglsConfig (sv.py:33-49),
SolveReport (sv.py:52-85), error_estimate / stopping_ratio (sv.py:88-117)
and pcgls (sv.py:120-268).  The whole loop -- products with A and A^T, the
preconditioner application, the dots, the scalar recursion, the delayed
error estimate and the stopping rule -- is device resident
(csrc/solver.cu): one captured CUDA graph per iteration, no host sync
inside it.  The returned iterate, iteration count, flags and ratio history
are bit-identical to the reference's.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .device import (BATCH, DeviceSolver, device_batch_solver, device_matrix, device_preconditioner,
                     device_solver, device_solvers)


@dataclass
class CglsConfig:
    """Solver controls; norm_A is the caller's spectral-norm estimate."""

    norm_A: float
    delta: float = 1e-10
    max_iters: int = 2000
    estimator_delay: int = 5
    ratio_raw: bool = False

    def __post_init__(self):
        if self.delta <= 0.0:
            raise ValueError("delta must be > 0")
        if self.estimator_delay < 1:
            raise ValueError("estimator_delay must be >= 1")
        if self.max_iters < 1:
            raise ValueError("max_iters must be >= 1")


@dataclass
class SolveReport:
    """Outcome of one pcgls run (fields and to_dict keys as sv.py:52-85)."""

    its: int
    converged: bool
    breakdown: bool
    ratio_pt_final: float
    ratio_pt_history: list = field(default_factory=list)
    psize: int = 0
    nmod: int = 0
    residual_norm_final: float = 0.0
    gradient_norm_final: float = 0.0

    def to_dict(self) -> dict:
        return {
            "its": self.its,
            "converged": self.converged,
            "breakdown": self.breakdown,
            "ratio_pt": self.ratio_pt_final,
            "ratio_pt_history": list(self.ratio_pt_history),
            "psize": self.psize,
            "nmod": self.nmod,
            "residual_norm": self.residual_norm_final,
            "gradient_norm": self.gradient_norm_final,
        }


def error_estimate(window, d) -> float:
    """Sum of the last d step decrements alpha_k * rho_k (sv.py:88-101)."""
    if d < 1:
        raise ValueError("d must be >= 1")
    window = list(window)
    if len(window) < d:
        raise ValueError("estimate not yet defined: fewer than d iterations available")
    return float(sum(a * r for a, r in window[-d:]))


def stopping_ratio(estim, norm_A, x_norm, b_norm, raw=False) -> float:
    """sqrt(estim) / (||A|| ||x|| + ||b||), or estim / (...) when raw (sv.py:104-117)."""
    denom = norm_A * x_norm + b_norm
    if denom <= 0.0:
        raise ValueError("zero denominator in stopping ratio")
    if estim < 0.0:
        estim = 0.0
    num = estim if raw else np.sqrt(estim)
    return float(num / denom)


def pcgls(A, b, pre, cfg: CglsConfig, iterate_hook=None):
    """Left-preconditioned CGLS from a zero start (sv.py:120-268).

    pre=None is plain CGLS.  iterate_hook(k, x) is supported on a slow path
    that returns x to the host after every iteration (tests only); without
    it the solve is one device loop with a 4-byte status poll per batch.
    Returns (x, SolveReport).
    """
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (int(A.nrows),):
        raise ValueError("right-hand side length mismatch")
    n = int(A.ncols)
    if pre is not None:
        if pre.factors.nrows != int(A.nrows) or pre.n != n:
            raise ValueError("preconditioner does not match the matrix")
        psize, nmod = pre.psize, pre.factors.nmod
    else:
        psize, nmod = 0, 0

    dA = device_matrix(A)
    dpre = device_preconditioner(pre, dA.ctx) if pre is not None else None
    solver = device_solver(dA, dpre)
    ccfg = solver.cfg_struct(cfg.norm_A, cfg.delta, cfg.max_iters, cfg.estimator_delay, cfg.ratio_raw)
    b = np.ascontiguousarray(b)
    x = np.empty(n)
    status = solver.start(L.ptr(b), L.RSB_HOST, ccfg)
    if status == 0:
        if iterate_hook is None:
            solver.iterate(cfg.max_iters)
        else:
            last = 0
            while True:
                it, st = solver.iterate(1)
                if it > last:
                    last = it
                    xi = np.empty(n)
                    solver.get_x(L.ptr(xi), L.RSB_HOST)
                    iterate_hook(it, xi)
                if st != 0:
                    break
    rep, hist = solver.finish(cfg.max_iters + cfg.estimator_delay + 2)
    solver.get_x(L.ptr(x), L.RSB_HOST)
    return x, _report(rep, hist, psize, nmod)


def _report(rep, hist, psize, nmod) -> SolveReport:
    return SolveReport(
        its=int(rep.its),
        converged=bool(rep.converged),
        breakdown=bool(rep.breakdown),
        ratio_pt_final=float(rep.ratio_pt_final),
        ratio_pt_history=[float(v) for v in hist],
        psize=psize,
        nmod=nmod,
        residual_norm_final=float(rep.residual_norm),
        gradient_norm_final=float(rep.gradient_norm),
    )


def _check(A, pre, m):
    n = int(A.ncols)
    if pre is not None:
        if pre.factors.nrows != int(A.nrows) or pre.n != n:
            raise ValueError("preconditioner does not match the matrix")
        return pre.psize, pre.factors.nmod
    return 0, 0


def pcgls_batch(A, B, pre, cfg: CglsConfig, streams: int | None = None):
    """Independent pcgls solves of A x_j ~ B[j] sharing A and pre (config 4's
    batch of right-hand sides per GPU).

    Not in the reference API: the reference solves one b per pcgls call; the
    result for each row of B is exactly pcgls(A, B[j], pre, cfg), bit for
    bit.  When the triangular solves are wide (grid schedules) and the
    coupling is cg / identity with the implicit Y, groups of 8 right-hand
    sides run through the batched kernels (csrc/bsolver.cu: every matrix and
    factor entry read once per group).  Otherwise -- or with `streams` given,
    or RSB_BATCH=streams -- each solve has its own CUDA stream and workspace
    over the one device copy of A and the factors, `streams` of them per
    library call (default: all); single-CTA solves (narrow DAGs, one SM each)
    then iterate all at once.  Returns (X with rows x_j, [reports]).
    """
    B = np.ascontiguousarray(np.atleast_2d(np.asarray(B, dtype=np.float64)))
    m, n = int(A.nrows), int(A.ncols)
    if B.ndim != 2 or B.shape[1] != m:
        raise ValueError("right-hand side length mismatch")
    psize, nmod = _check(A, pre, m)
    k = B.shape[0]
    X = np.empty((k, n))
    reports: list[SolveReport] = []
    if k == 0:
        return X, reports
    dA = device_matrix(A)
    dpre = device_preconditioner(pre, dA.ctx) if pre is not None else None
    mode = os.environ.get("RSB_BATCH", "auto")
    bs = device_batch_solver(dA, dpre) if (mode != "streams" and streams is None) else None
    if bs is not None:
        # kernels that serve 8 right-hand sides per pass (csrc/bsolver.cu)
        ccfg = DeviceSolver.cfg_struct(cfg.norm_A, cfg.delta, cfg.max_iters, cfg.estimator_delay, cfg.ratio_raw)
        cap = cfg.max_iters + cfg.estimator_delay + 2
        for lo in range(0, k, BATCH):
            c = min(BATCH, k - lo)
            Bc = np.ascontiguousarray(B[lo:lo + c])
            reps = (L.ReportC * c)()
            hist = np.empty((c, cap))
            Xc = np.empty((c, n))
            L.check(L.lib().rsb_pcgls_batch8(bs.h, c, L.ptr(Bc), L.RSB_HOST, ctypes.byref(ccfg), L.ptr(Xc), reps,
                                             L.ptr(hist), cap))
            X[lo:lo + c] = Xc
            for i in range(c):
                reports.append(_report(reps[i], hist[i, : min(reps[i].history_len, cap)].copy(), psize, nmod))
        return X, reports
    width = k if streams is None else max(1, min(int(streams), k))
    solvers = device_solvers(dA, dpre, width)
    ccfg = DeviceSolver.cfg_struct(cfg.norm_A, cfg.delta, cfg.max_iters, cfg.estimator_delay, cfg.ratio_raw)
    cap = cfg.max_iters + cfg.estimator_delay + 2
    for lo in range(0, k, width):
        c = min(width, k - lo)
        hs = (ctypes.c_void_p * c)(*[s.h for s in solvers[:c]])
        bs = (ctypes.c_void_p * c)(*[B[lo + i].ctypes.data for i in range(c)])
        xs = (ctypes.c_void_p * c)(*[X[lo + i].ctypes.data for i in range(c)])
        reps = (L.ReportC * c)()
        hist = np.empty((c, cap))
        L.check(L.lib().rsb_pcgls_many(c, hs, bs, L.RSB_HOST, ctypes.byref(ccfg), xs, reps, L.ptr(hist), cap))
        for i in range(c):
            reports.append(_report(reps[i], hist[i, : min(reps[i].history_len, cap)].copy(), psize, nmod))
    return X, reports
