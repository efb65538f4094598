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

from dataclasses import dataclass, field

import numpy as np

from . import _lib as L
from .device import device_matrix, device_preconditioner, device_solver


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
    report = SolveReport(
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
    return x, report
