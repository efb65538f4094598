"""Host logic of the row-partitioned pcgls (paper_2603_28642_b200/distributed.py)
on CPU: gloo, world sizes 1, 2 and 4.

The ranks use gloo and a CPU compute backend built on the oracle kernels
(test infrastructure) with the DeviceBackend's interface.  One rank
reproduces the single-device pcgls bit for bit (every local order is the
global order); more ranks re-associate q.q, the s-dots and the A^T / L2^T
sums across row blocks -- in rank order, so the result is deterministic --
and must agree to rounding and take the same number of iterations.
"""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_28642_b200 import distributed as D


class CpuBackend:
    """DeviceBackend's interface on the oracle kernels (torch CPU tensors)."""

    def __init__(self):
        import torch

        self.torch = torch

    def matrix(self, M):
        return M

    def array(self, a):
        return self.torch.tensor(np.asarray(a, dtype=np.float64))

    def index(self, a):
        return self.torch.as_tensor(np.asarray(a, dtype=np.int64))

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64)

    def to_host(self, t):
        return t.numpy().copy()

    def matvec(self, M, x):
        return self.torch.from_numpy(O.matvec(M, x.numpy()))

    def matvec_t(self, M, y):
        return self.torch.from_numpy(O.matvec_transpose(M, y.numpy()))

    def solve(self, T, kind, b):
        b = b.numpy()
        if kind == 1:
            return self.torch.from_numpy(O.sparse_lower_solve(T, b, unit_diag=True))
        if kind == 4:
            return self.torch.from_numpy(O.sparse_lower_solve_transpose(T, b, unit_diag=True))
        return self.torch.from_numpy(O.sparse_upper_solve(T, b))

    def dot(self, a, b):
        return self.torch.tensor([O.dot(a.numpy(), b.numpy())], dtype=self.torch.float64)

    def axpy(self, y, alpha, x):
        return self.torch.add(y, self.torch.mul(x, alpha))

    def axmy(self, y, alpha, x):
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


class SingleComm:
    rank, world = 0, 1

    def sum_(self, t):
        return t

    def sum_scalar(self, t):
        return float(t.item())

    def allgather_padded(self, t, width):
        import torch

        buf = torch.zeros(width, dtype=t.dtype)
        buf[: t.numel()] = t
        return [buf]


def problem(mode="cg"):
    import paper_2603_28642_b200 as P
    from paper_2603_28642_b200 import workloads as W

    A, b = W.config0(seed=3, m=450, n=300)
    S, _ = P.column_scale(A)
    na = O.power_method_norm2(S, 100, 3)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=1e-3, mu=1.0))
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
    cfg = P.CglsConfig(norm_A=na, delta=1e-8, max_iters=40)
    return S, b, pre, cfg, na


def test_row_blocks_cover_rows():
    for m, w in [(10, 3), (7, 7), (98304, 8), (1, 1)]:
        blocks = D.row_blocks(m, w)
        assert blocks[0][0] == 0 and blocks[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
        assert max(h - l for l, h in blocks) - min(h - l for l, h in blocks) <= 1


def test_partition_owns_every_row_once():
    S, b, pre, cfg, na = problem()
    perm = pre.factors.row_perm.perm
    for w in (1, 2, 3, 4):
        P_ = D.Partition(S.nrows, S.ncols, perm, w)
        assert np.array_equal(np.sort(np.concatenate(P_.r1_pos)), np.arange(S.ncols))
        assert np.array_equal(np.sort(np.concatenate(P_.l2_rows)), np.arange(S.nrows - S.ncols))
        for g, (lo, hi) in enumerate(P_.blocks):
            assert np.array_equal(perm[P_.r1_pos[g]], lo + P_.r1_local[g])
            assert np.array_equal(perm[S.ncols + P_.l2_rows[g]], lo + P_.r2_local[g])


def test_local_products_sum_to_global():
    S, b, pre, cfg, na = problem()
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal(S.ncols), rng.standard_normal(S.nrows)
    blocks = D.row_blocks(S.nrows, 3)
    parts = [D.local_rows(S, lo, hi) for lo, hi in blocks]
    assert np.array_equal(np.concatenate([O.matvec(P_, x) for P_ in parts]), O.matvec(S, x))
    zsum = sum(O.matvec_transpose(P_, y[lo:hi]) for P_, (lo, hi) in zip(parts, blocks))
    assert np.allclose(zsum, O.matvec_transpose(S, y), rtol=1e-13, atol=1e-13)
    # L2 rows selected by owner keep the global column order: one block is L2 itself
    L2 = pre.factors.L2
    sel = D.select_rows(L2, np.arange(L2.nrows))
    assert np.array_equal(O.matvec_transpose(sel, y[: L2.nrows]), O.matvec_transpose(L2, y[: L2.nrows]))


@pytest.mark.parametrize("mode", ["cg", "identity"])
def test_single_rank_is_bitwise_pcgls(mode):
    S, b, pre, cfg, na = problem(mode)
    x1, rep1 = D.pcgls_row_partitioned(S, b, pre, cfg, SingleComm(), CpuBackend())
    xo, repo = O.pcgls(S, b, O.OraclePreconditioner.from_reference(pre), na, delta=cfg.delta,
                       max_iters=cfg.max_iters)
    assert np.array_equal(x1, xo)
    assert rep1.its == repo["its"] and rep1.converged == repo["converged"]
    assert rep1.ratio_pt_history == repo["ratio_pt_history"]
    assert rep1.residual_norm_final == repo["residual_norm"]
    assert rep1.gradient_norm_final == repo["gradient_norm"]


def test_dense_coupling_rejected():
    S, b, pre, cfg, na = problem("dense")
    with pytest.raises(ValueError):
        D.pcgls_row_partitioned(S, b, pre, cfg, SingleComm(), CpuBackend())


def _worker(rank, world, port, out, mode):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S, b, pre, cfg, na = problem(mode)
        comm = D.TorchComm()
        x, rep = D.pcgls_row_partitioned(S, b, pre, cfg, comm, CpuBackend())
        x2, rep2 = D.pcgls_row_partitioned(S, b, pre, cfg, comm, CpuBackend())
        assert np.array_equal(x, x2) and rep.ratio_pt_history == rep2.ratio_pt_history  # deterministic
        np.save(out.replace(".npy", f"_{rank}.npy"),
                np.concatenate([[rep.its, rep.converged, rep.residual_norm_final], x]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("mode", ["cg", "identity"])
def test_multi_rank_gloo_matches_single(tmp_path, world, mode):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "r.npy")
    mp.start_processes(_worker, args=(world, port, out, mode), nprocs=world, join=True, start_method="spawn")
    got = [np.load(out.replace(".npy", f"_{r}.npy")) for r in range(world)]
    for g in got[1:]:
        assert np.array_equal(g, got[0]), "ranks disagree"
    S, b, pre, cfg, na = problem(mode)
    x1, rep1 = D.pcgls_row_partitioned(S, b, pre, cfg, SingleComm(), CpuBackend())
    assert int(got[0][0]) == rep1.its and bool(got[0][1]) == rep1.converged
    assert abs(got[0][2] - rep1.residual_norm_final) <= 1e-10 * rep1.residual_norm_final
    x2 = got[0][3:]
    assert np.linalg.norm(x2 - x1) <= 1e-10 * np.linalg.norm(x1)
