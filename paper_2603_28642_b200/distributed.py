"""Row-partitioned single-RHS pcgls across ranks (second mode).

The m rows of A are split into contiguous blocks, one per rank.  Per iteration
(mirroring sv.py:202-241):

  q_g = A_g p                     local rows, no communication
  q.q = allreduce(q_g . q_g)      one scalar allreduce
  x += alpha p ; r_g -= alpha q_g x replicated, r row-partitioned
  z = allreduce(A_g^T r_g)        one allreduce of the n-vector per A^T product
  r = allgather(r_g)              the apply needs r in pivot order (pc.py:159-161)
  h = apply(r)                    replicated factors, replicated apply
  z.z, z.h, z.p, ||x||            replicated n-vector dots (exact order)

Every rank carries the same scalar state, so every branch of the reference
(sv.py:203-241, 243-253) is taken identically on all ranks.  With one rank the
arithmetic is the single-GPU pcgls's, bit for bit; with more ranks the sums
behind q.q and A^T r are re-associated across row blocks (documented in
DESIGN.md; tests bound the difference and require the same iteration count).

Communication and local compute are pluggable: `TorchComm` wraps
torch.distributed (NCCL on GPUs, gloo on CPUs) and `DeviceBackend` runs the
local products, the apply and the dots through librowsplit_b200.so on device
tensors.  Tests inject a CPU backend to cover the host logic with gloo.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .types import CscMatrix


def row_blocks(m: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, balanced row blocks [lo, hi) for each rank."""
    base, extra = divmod(m, world)
    out, lo = [], 0
    for g in range(world):
        hi = lo + base + (1 if g < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


def local_rows(A, lo: int, hi: int) -> CscMatrix:
    """Rows lo..hi-1 of a CSC matrix, as an (hi-lo) x n CSC matrix (row
    indices shifted, column order and within-column row order preserved)."""
    A = CscMatrix.of(A)
    keep = (A.row_idx >= lo) & (A.row_idx < hi)
    cols = np.repeat(np.arange(A.ncols, dtype=np.int64), A.column_counts())[keep]
    col_ptr = np.zeros(A.ncols + 1, dtype=np.int64)
    if len(cols):
        col_ptr[1:] = np.cumsum(np.bincount(cols, minlength=A.ncols))
    return CscMatrix(hi - lo, A.ncols, col_ptr, A.row_idx[keep] - lo, A.values[keep])


@dataclass
class PartitionedReport:
    its: int
    converged: bool
    breakdown: bool
    ratio_pt_final: float
    ratio_pt_history: list
    residual_norm_final: float
    gradient_norm_final: float
    iters_run: int


class TorchComm:
    """torch.distributed collectives on vectors of the backend's array type."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device

    def allreduce_(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t

    def allreduce_scalar(self, v: float) -> float:
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.device)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return float(t.item())

    def allgather_cat(self, t, sizes):
        parts = [self.torch.empty(s, dtype=t.dtype, device=t.device) for s in sizes]
        self.dist.all_gather(parts, t.contiguous())
        return self.torch.cat(parts)


class DeviceBackend:
    """Local compute on one GPU: products, apply and exact-order dots through
    librowsplit_b200.so on torch CUDA tensors (device pointers, where=DEVICE)."""

    def __init__(self, A_local, pre, device_index: int):
        import torch

        from . import _lib as L
        from .device import DeviceMatrix, device_preconditioner, get_context

        self.torch, self.L = torch, L
        self.dev = torch.device("cuda", device_index)
        self.ctx = get_context(device_index)
        self.A = DeviceMatrix(A_local, self.ctx)
        self.pre = device_preconditioner(pre, self.ctx) if pre is not None else None

    def array(self, a):
        return self.torch.as_tensor(np.asarray(a, dtype=np.float64), device=self.dev).contiguous()

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.dev)

    def to_host(self, t):
        return t.detach().cpu().numpy()

    def _sync(self):
        self.torch.cuda.synchronize(self.dev)

    def matvec(self, x):
        y = self.zeros(self.A.nrows)
        self._sync()
        self.L.check(self.L.lib().rsb_matvec(self.A.h, x.data_ptr(), y.data_ptr(), self.L.RSB_DEVICE))
        return y

    def matvec_t(self, y):
        z = self.zeros(self.A.ncols)
        self._sync()
        self.L.check(self.L.lib().rsb_matvec_transpose(self.A.h, y.data_ptr(), z.data_ptr(), self.L.RSB_DEVICE))
        return z

    def apply(self, r1, r2):
        h = self.zeros(self.pre.n)
        r1, r2 = r1.contiguous(), r2.contiguous()
        self._sync()
        self.L.check(self.L.lib().rsb_pre_apply(self.pre.h, r1.data_ptr(), r2.data_ptr(), h.data_ptr(),
                                                self.L.RSB_DEVICE))
        return h

    def dot(self, a, b) -> float:
        out = np.zeros(1)
        self._sync()
        self.L.check(self.L.lib().rsb_dot(self.ctx.h, a.numel(), a.data_ptr(), b.data_ptr(),
                                          out.ctypes.data_as(self.L.f64p), self.L.RSB_DEVICE))
        return float(out[0])

    # elementwise updates: one rounding for the product, one for the sum
    def axpy(self, y, alpha, x):  # y + alpha * x
        return self.torch.add(y, self.torch.mul(x, alpha))

    def axmy(self, y, alpha, x):  # y - alpha * x
        return self.torch.sub(y, self.torch.mul(x, alpha))

    def take(self, v, idx):
        return v[self.torch.as_tensor(idx, device=self.dev)]

    def sub(self, a, b):
        return self.torch.sub(a, b)


def pcgls_row_partitioned(A, b, pre, cfg, comm, make_backend):
    """Row-partitioned pcgls.  A, b, pre are the global problem (identical on
    every rank); each rank keeps its row block of A and b.  make_backend(A_local,
    pre) builds the rank's local compute.  Returns (x as host array, report)."""
    m, n = int(A.nrows), int(A.ncols)
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (m,):
        raise ValueError("right-hand side length mismatch")
    blocks = row_blocks(m, comm.world)
    lo, hi = blocks[comm.rank]
    sizes = [h - l for l, h in blocks]
    A_local = local_rows(A, lo, hi)
    be = make_backend(A_local, pre)
    d = cfg.estimator_delay
    perm = np.asarray(pre.factors.row_perm.perm) if pre is not None else None

    b_l = be.array(b[lo:hi])
    b_norm = math.sqrt(comm.allreduce_scalar(be.dot(b_l, b_l)))

    def grad(r_l):
        z = be.matvec_t(r_l)
        return comm.allreduce_(z)

    def precondition(r_l, z):
        if pre is None:
            return z.clone()
        r = comm.allgather_cat(r_l, sizes)
        return be.apply(be.take(r, perm[:n]), be.take(r, perm[n:]))

    x = be.zeros(n)
    r_l = b_l.clone()
    z = grad(r_l)
    zz = be.dot(z, z)
    alphas, sigmas, x_norms, history = [], [], [0.0], []
    converged, stopped, its_cert, iters_run = False, False, 0, 0
    if zz == 0.0:
        return be.to_host(x), PartitionedReport(0, True, False, 0.0, [0.0], b_norm, 0.0, 0)
    h = precondition(r_l, z)
    rho = be.dot(z, h)
    p = h.clone()
    for it in range(cfg.max_iters):
        sigma = rho if rho > 0.0 else be.dot(z, p)
        if sigma == 0.0:
            p = z.clone()
            sigma = zz
            rho = sigma
        q_l = be.matvec(p)
        qq = comm.allreduce_scalar(be.dot(q_l, q_l))
        if qq <= 0.0 or sigma == 0.0:
            stopped = True
            break
        alpha = sigma / qq
        x = be.axpy(x, alpha, p)
        r_l = be.axmy(r_l, alpha, q_l)
        alphas.append(alpha)
        sigmas.append(sigma)
        x_norms.append(math.sqrt(be.dot(x, x)))
        iters_run = it + 1
        i = iters_run - d
        if i >= 0:
            ratio = _ratio(alphas, sigmas, i, cfg, x_norms[i], b_norm)
            history.append(ratio)
            if ratio <= cfg.delta:
                converged, its_cert = True, i
                break
        z = grad(r_l)
        zz = be.dot(z, z)
        if zz == 0.0:
            stopped = True
            break
        h = precondition(r_l, z)
        rho_new = be.dot(z, h)
        p = be.axpy(h, rho_new / rho, p) if rho != 0.0 else h.clone()
        rho = rho_new
    if stopped and not converged:
        for i in range(max(0, iters_run - d + 1), iters_run + 1):
            ratio = _ratio(alphas, sigmas, i, cfg, x_norms[i], b_norm)
            history.append(ratio)
            if ratio <= cfg.delta:
                converged, its_cert = True, i
                break
    fr_l = be.sub(b_l, be.matvec(x))
    res = math.sqrt(comm.allreduce_scalar(be.dot(fr_l, fr_l)))
    g = grad(fr_l)
    rep = PartitionedReport(its_cert if converged else iters_run, converged, stopped and not converged,
                            history[-1] if history else float("inf"), history, res,
                            math.sqrt(be.dot(g, g)), iters_run)
    return be.to_host(x), rep


def _ratio(alphas, sigmas, i, cfg, x_norm, b_norm):
    """error_estimate + stopping_ratio (sv.py:88-117): Python's compensated sum
    of the window, sqrt (unless raw), over ||A|| ||x_i|| + ||b||."""
    estim = float(sum(a * s for a, s in zip(alphas[i:], sigmas[i:])))
    denom = cfg.norm_A * x_norm + b_norm
    if denom <= 0.0:
        raise ValueError("zero denominator in stopping ratio")
    if estim < 0.0:
        estim = 0.0
    num = estim if cfg.ratio_raw else math.sqrt(estim)
    return float(num / denom)
