"""Row-partitioned single-RHS pcgls across ranks (second mode).

The m rows of A are split into contiguous blocks of original rows, one per
rank; a rank also owns the rows of L2 whose original row is in its block
(L2's row i is pivot position n + i, original row perm[n + i]), so the
coupling system's vectors are partitioned with them.  x, p, z, h and the
factors L1 and U are replicated: the triangular solves run redundantly on
every rank (they cannot be split without per-level communication).  Per
iteration (sv.py:202-241; pc.py:135-186, 284-310):

  q_g = A_g p                      local rows
  q.q = sum_g q_g.q_g              scalar partials, summed in rank order
  x += alpha p ; r_g -= alpha q_g  (x replicated, r row-partitioned)
  z = sum_g A_g^T r_g              the n-vector exchange of the A^T product
  r1 = r[perm[:n]]                 an all-gather of each rank's r1 entries
  t1 = L1^-1 r1; u_g = r2_g - L2_g t1
  inner CG on S: its s-vectors partitioned, one n-vector exchange per
  L2^T product (L2_g^T w_g summed over ranks), s-dots summed in rank order
  h = U^-1 L1^-1 (r1 + L1^-T L2^T w)   replicated

Every rank carries the same scalars, so every branch of the reference is
taken identically everywhere.  With one rank the arithmetic is the
single-GPU pcgls's, bit for bit (local orders are the global orders); with
more ranks the sums behind q.q, the s-dots and the A^T / L2^T products are
re-associated across row blocks -- in rank order, deterministically
(reduce="ordered", an all-gather of the partials) or by NCCL's all-reduce
(reduce="nccl", fewer bytes).

Communication and local compute are pluggable: `TorchComm` wraps
torch.distributed (NCCL on GPUs, gloo on CPUs); `DeviceBackend` runs the
products, solves and dots through librowsplit_b200.so on the context's CUDA
stream (RSB_DEVICE_ASYNC: no host synchronisation inside an operation) with
torch's elementwise updates and the collectives ordered on the same
stream.  Tests inject a CPU backend to cover the host logic with gloo.
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


def select_rows(A, rows) -> CscMatrix:
    """The rows `rows` (original ids, in the order wanted locally) of a CSC
    matrix as a len(rows) x n CSC matrix.  Entries keep their original
    order inside each column, so column sums run in the global order."""
    A = CscMatrix.of(A)
    rows = np.asarray(rows, dtype=np.int64)
    inv = np.full(A.nrows, -1, dtype=np.int64)
    inv[rows] = np.arange(len(rows), dtype=np.int64)
    new = inv[A.row_idx]
    keep = new >= 0
    cols = np.repeat(np.arange(A.ncols, dtype=np.int64), A.column_counts())[keep]
    col_ptr = np.zeros(A.ncols + 1, dtype=np.int64)
    if len(cols):
        col_ptr[1:] = np.cumsum(np.bincount(cols, minlength=A.ncols))
    return CscMatrix(len(rows), A.ncols, col_ptr, new[keep], A.values[keep])


def local_rows(A, lo: int, hi: int) -> CscMatrix:
    """Rows lo..hi-1 of a CSC matrix (row indices shifted)."""
    return select_rows(A, np.arange(lo, hi, dtype=np.int64))


class Partition:
    """Who owns what.  Rank g: original rows [lo_g, hi_g) of A and b; the r1
    entries i (pivot positions < n) whose original row perm[i] it owns, in
    increasing i; its L2 rows (positions n + i with perm[n + i] owned), in
    increasing i."""

    def __init__(self, m: int, n: int, perm, world: int):
        self.m, self.n, self.world = m, n, world
        self.blocks = row_blocks(m, world)
        perm = np.asarray(perm, dtype=np.int64) if perm is not None else None
        self.owner_of_row = np.empty(m, dtype=np.int64)
        for g, (lo, hi) in enumerate(self.blocks):
            self.owner_of_row[lo:hi] = g
        if perm is None:
            return
        own1 = self.owner_of_row[perm[:n]]
        own2 = self.owner_of_row[perm[n:]]
        # per rank: r1 positions and their local row index; L2 rows and the
        # local row index of their residual entry
        self.r1_pos = [np.flatnonzero(own1 == g) for g in range(world)]
        self.r1_local = [perm[p] - self.blocks[g][0] for g, p in enumerate(self.r1_pos)]
        self.l2_rows = [np.flatnonzero(own2 == g) for g in range(world)]
        self.r2_local = [perm[n + i] - self.blocks[g][0] for g, i in enumerate(self.l2_rows)]
        self.r1_max = max(len(p) for p in self.r1_pos)


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
    """torch.distributed collectives on the backend's tensors.

    reduce="ordered": sums of per-rank partials are formed by an all-gather
    and added in rank order (deterministic for a given world size);
    reduce="nccl": all_reduce."""

    def __init__(self, device=None, reduce: str = "ordered"):
        import torch
        import torch.distributed as dist

        if reduce not in ("ordered", "nccl"):
            raise ValueError("reduce must be 'ordered' or 'nccl'")
        self.torch, self.dist = torch, dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        self.device = device
        self.reduce = reduce

    def sum_(self, t):
        """in-place sum over ranks of a tensor (vector or 1-element)"""
        if self.world == 1:
            return t
        if self.reduce == "nccl":
            self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
            return t
        parts = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t.contiguous())
        acc = parts[0]
        for q in parts[1:]:
            acc = self.torch.add(acc, q)
        t.copy_(acc)
        return t

    def sum_scalar(self, t) -> float:
        """rank-ordered sum of 1-element partials, read on the host"""
        if self.world > 1:
            parts = [self.torch.empty_like(t) for _ in range(self.world)]
            self.dist.all_gather(parts, t.contiguous())
            acc = parts[0]
            for q in parts[1:]:
                acc = self.torch.add(acc, q)
            t = acc
        return float(t.item())

    def allgather_padded(self, t, width):
        """every rank's t (length <= width, zero-padded) -> list of tensors"""
        buf = self.torch.zeros(width, dtype=t.dtype, device=t.device)
        buf[: t.numel()] = t
        if self.world == 1:
            return [buf]
        parts = [self.torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(parts, buf)
        return parts


class DeviceBackend:
    """Local compute on one GPU through librowsplit_b200.so: every product,
    solve and dot is enqueued on the context's stream (RSB_DEVICE_ASYNC),
    which is also torch's current stream for the elementwise updates and the
    collectives, so nothing inside an operation waits on the host."""

    def __init__(self, device_index: int):
        import ctypes

        import torch

        from . import _lib as L
        from .device import get_context

        self.torch, self.L = torch, L
        self.dev = torch.device("cuda", device_index)
        self.ctx = get_context(device_index)
        h = ctypes.c_void_p()
        L.check(L.lib().rsb_ctx_stream(self.ctx.h, ctypes.byref(h)))
        self.stream = torch.cuda.ExternalStream(h.value, device=self.dev)

    def stream_context(self):
        return self.torch.cuda.stream(self.stream)

    def matrix(self, M):
        from .device import DeviceMatrix

        return DeviceMatrix(M, self.ctx)

    def array(self, a):
        return self.torch.as_tensor(np.asarray(a, dtype=np.float64), device=self.dev).contiguous()

    def index(self, a):
        return self.torch.as_tensor(np.asarray(a, dtype=np.int64), device=self.dev)

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.dev)

    def to_host(self, t):
        return t.detach().cpu().numpy()

    def matvec(self, dM, x):
        y = self.torch.empty(dM.nrows, dtype=self.torch.float64, device=self.dev)
        if dM.nrows:
            self.L.check(self.L.lib().rsb_matvec(dM.h, x.data_ptr(), y.data_ptr(), self.L.RSB_DEVICE_ASYNC))
        return y

    def matvec_t(self, dM, y):
        z = self.torch.empty(dM.ncols, dtype=self.torch.float64, device=self.dev)
        self.L.check(self.L.lib().rsb_matvec_transpose(dM.h, y.data_ptr() if y.numel() else None, z.data_ptr(),
                                                       self.L.RSB_DEVICE_ASYNC))
        return z

    def solve(self, dT, kind, b):
        x = self.torch.empty(dT.ncols, dtype=self.torch.float64, device=self.dev)
        self.L.check(self.L.lib().rsb_trsv(dT.h, kind, b.data_ptr(), x.data_ptr(), self.L.RSB_DEVICE_ASYNC))
        return x

    def dot(self, a, b):
        """a @ b in the reference's order, as a 1-element device tensor"""
        out = self.torch.empty(1, dtype=self.torch.float64, device=self.dev)
        if a.numel() == 0:
            out.zero_()
            return out
        import ctypes

        self.L.check(self.L.lib().rsb_dot(self.ctx.h, a.numel(), a.data_ptr(), b.data_ptr(),
                                          ctypes.cast(out.data_ptr(), self.L.f64p), self.L.RSB_DEVICE_ASYNC))
        return out

    # elementwise updates: one rounding for the product, one for the sum
    def axpy(self, y, alpha, x):  # y + alpha * x
        return self.torch.add(y, self.torch.mul(x, alpha))

    def axmy(self, y, alpha, x):  # y - alpha * x
        return self.torch.sub(y, self.torch.mul(x, alpha))

    def add(self, a, b):
        return self.torch.add(a, b)

    def sub(self, a, b):
        return self.torch.sub(a, b)

    def take(self, v, idx):
        return v[idx]

    def scatter_into(self, out, idx, vals):
        out[idx] = vals
        return out


TRI_LOWER_UNIT, TRI_UPPER, TRI_LOWER_T_UNIT = 1, 2, 4


class RowPartition:
    """The rank's share of the problem on its backend: its row block of A,
    its rows of L2, the replicated L1 and U, the index maps of the r1
    exchange.  Built once (uploads and analyses), reused by every solve."""

    def __init__(self, A, pre, comm, be):
        m, n = int(A.nrows), int(A.ncols)
        self.m, self.n, self.comm, self.be = m, n, comm, be
        self.pre = pre
        perm = pre.factors.row_perm.perm if pre is not None else None
        self.part = Partition(m, n, perm, comm.world)
        g = comm.rank
        lo, hi = self.part.blocks[g]
        self.A = A
        self.dA = be.matrix(local_rows(A, lo, hi))
        self.lo, self.hi = lo, hi
        if pre is None:
            return
        f = pre.factors
        P = self.part
        self.s_l = len(P.l2_rows[g])
        self.dL1 = be.matrix(f.L1)
        self.dU = be.matrix(f.U)
        self.dL2 = be.matrix(select_rows(f.L2, P.l2_rows[g]))
        self.r1_local = be.index(P.r1_local[g])
        self.r2_local = be.index(P.r2_local[g])
        self.r1_pos = [be.index(p) for p in P.r1_pos]
        self.mode = getattr(pre.s_mode, "value", pre.s_mode)
        if getattr(pre.y_mode, "value", pre.y_mode) != "implicit" or self.mode == "dense":
            raise ValueError("the row-partitioned solve needs the implicit Y with cg or identity coupling")

    def gather_r1(self, r_l):
        """r1 = r[perm[:n]] from every rank's entries (pure data movement)"""
        be = self.be
        parts = self.comm.allgather_padded(be.take(r_l, self.r1_local), self.part.r1_max)
        r1 = be.zeros(self.n)
        for g, pos in enumerate(self.r1_pos):
            if pos.numel():
                be.scatter_into(r1, pos, parts[g][: pos.numel()])
        return r1

    def l2t(self, w_l):
        """L2^T w = sum over ranks of L2_g^T w_g"""
        return self.comm.sum_(self.be.matvec_t(self.dL2, w_l))

    def s_matvec(self, p_l):
        """S p = p + L2 L1^-1 L1^-T L2^T p  (pc.py:149-154), p partitioned"""
        be = self.be
        a = self.l2t(p_l)
        bb = be.solve(self.dL1, TRI_LOWER_UNIT, be.solve(self.dL1, TRI_LOWER_T_UNIT, a))
        return be.add(p_l, be.matvec(self.dL2, bb))

    def sdot(self, a, b) -> float:
        return self.comm.sum_scalar(self.be.dot(a, b))

    def cg(self, u_l, iters):
        """_cg_fixed_steps (pc.py:284-310) with partitioned s-vectors"""
        be = self.be
        w = be.zeros(self.s_l)
        r = u_l.clone()
        rho = self.sdot(r, r)
        if rho == 0.0:
            return w
        p = r.clone()
        for _ in range(iters):
            q = self.s_matvec(p)
            pq = self.sdot(p, q)
            if pq <= 0.0:
                break
            alpha = rho / pq
            w = be.axpy(w, alpha, p)
            r = be.axmy(r, alpha, q)
            rho_new = self.sdot(r, r)
            if rho_new == 0.0:
                break
            p = be.axpy(r, rho_new / rho, p)
            rho = rho_new
        return w

    def precondition(self, r_l, z):
        """h = apply(r1, r2)  (pc.py:175-186)"""
        be = self.be
        if self.pre is None:
            return z.clone()
        r1 = self.gather_r1(r_l)
        if self.pre.factors.L2.nrows:
            r2 = be.take(r_l, self.r2_local)
            t1 = be.solve(self.dL1, TRI_LOWER_UNIT, r1)
            u = be.sub(r2, be.matvec(self.dL2, t1))
            w = u if self.mode == "identity" else self.cg(u, int(self.pre.cg_iters))
            y = be.add(r1, be.solve(self.dL1, TRI_LOWER_T_UNIT, self.l2t(w)))  # r1 + Y^T w, Y^T = L1^-T L2^T
        else:
            y = r1
        return be.solve(self.dU, TRI_UPPER, be.solve(self.dL1, TRI_LOWER_UNIT, y))


def pcgls_row_partitioned(A, b, pre, cfg, comm, backend, part: RowPartition | None = None):
    """Row-partitioned pcgls.  A, b, pre are the global problem (identical on
    every rank); each rank uses its share (`part`, built here when not
    given).  `backend` is the rank's local compute (DeviceBackend on a
    GPU).  Returns (x as host array, report)."""
    m, n = int(A.nrows), int(A.ncols)
    b = np.asarray(b, dtype=np.float64)
    if b.shape != (m,):
        raise ValueError("right-hand side length mismatch")
    be = backend
    ctx_mgr = be.stream_context() if hasattr(be, "stream_context") else None
    if ctx_mgr is not None:
        with ctx_mgr:
            ops = part if part is not None else RowPartition(A, pre, comm, be)
            return _pcgls(ops, b, pre, cfg, comm, be, n)
    ops = part if part is not None else RowPartition(A, pre, comm, be)
    return _pcgls(ops, b, pre, cfg, comm, be, n)


def _pcgls(ops, b, pre, cfg, comm, be, n):
    d = cfg.estimator_delay
    b_l = be.array(b[ops.lo:ops.hi])
    b_norm = math.sqrt(ops.sdot(b_l, b_l))

    def grad(r_l):
        return comm.sum_(be.matvec_t(ops.dA, r_l))

    def rdot(a, c):  # replicated n-vectors: no exchange
        return float(be.dot(a, c).item())

    x = be.zeros(n)
    r_l = b_l.clone()
    z = grad(r_l)
    zz = rdot(z, z)
    alphas, sigmas, x_norms, history = [], [], [0.0], []
    converged, stopped, its_cert, iters_run = False, False, 0, 0
    if zz == 0.0:
        return be.to_host(x), PartitionedReport(0, True, False, 0.0, [0.0], b_norm, 0.0, 0)
    h = ops.precondition(r_l, z)
    rho = rdot(z, h)
    p = h.clone()
    for it in range(cfg.max_iters):
        sigma = rho if rho > 0.0 else rdot(z, p)
        if sigma == 0.0:
            p = z.clone()
            sigma = zz
            rho = sigma
        q_l = be.matvec(ops.dA, p)
        qq = ops.sdot(q_l, q_l)
        if qq <= 0.0 or sigma == 0.0:
            stopped = True
            break
        alpha = sigma / qq
        x = be.axpy(x, alpha, p)
        r_l = be.axmy(r_l, alpha, q_l)
        alphas.append(alpha)
        sigmas.append(sigma)
        x_norms.append(math.sqrt(rdot(x, x)))
        iters_run = it + 1
        i = iters_run - d
        if i >= 0:
            ratio = _ratio(alphas, sigmas, i, cfg, x_norms[i], b_norm)
            history.append(ratio)
            if ratio <= cfg.delta:
                converged, its_cert = True, i
                break
        z = grad(r_l)
        zz = rdot(z, z)
        if zz == 0.0:
            stopped = True
            break
        h = ops.precondition(r_l, z)
        rho_new = rdot(z, h)
        p = be.axpy(h, rho_new / rho, p) if rho != 0.0 else h.clone()
        rho = rho_new
    if stopped and not converged:
        for i in range(max(0, iters_run - d + 1), iters_run + 1):
            ratio = _ratio(alphas, sigmas, i, cfg, x_norms[i], b_norm)
            history.append(ratio)
            if ratio <= cfg.delta:
                converged, its_cert = True, i
                break
    fr_l = be.sub(b_l, be.matvec(ops.dA, x))
    res = math.sqrt(ops.sdot(fr_l, fr_l))
    gfin = grad(fr_l)
    rep = PartitionedReport(its_cert if converged else iters_run, converged, stopped and not converged,
                            history[-1] if history else float("inf"), history, res,
                            math.sqrt(rdot(gfin, gfin)), iters_run)
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
