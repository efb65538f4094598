"""Host logic of the multi-rank paths on CPU (gloo, world size 2).

The row-partitioned pcgls (paper_2603_28642_b200/distributed.py) runs its
collectives through torch.distributed; on this CPU-only container the ranks
use gloo and a CPU compute backend built on the oracle kernels (test
infrastructure).  One rank reproduces the single-device pcgls bit for bit;
two ranks re-associate q.q and A^T r across row blocks, so they must agree
to rounding and take the same number of iterations.
"""

import os

import numpy as np
import pytest

from oracle import oracle as O
from paper_2603_28642_b200 import distributed as D


class CpuBackend:
    def __init__(self, A_local, pre):
        import torch

        self.torch = torch
        self.A = A_local
        self.op = O.OraclePreconditioner.from_reference(pre) if pre is not None else None

    def array(self, a):
        return self.torch.tensor(np.asarray(a, dtype=np.float64))

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64)

    def to_host(self, t):
        return t.numpy().copy()

    def matvec(self, x):
        return self.torch.from_numpy(O.matvec(self.A, x.numpy()))

    def matvec_t(self, y):
        return self.torch.from_numpy(O.matvec_transpose(self.A, y.numpy()))

    def apply(self, r1, r2):
        return self.torch.from_numpy(self.op.apply(r1.numpy(), r2.numpy()))

    def dot(self, a, b):
        return O.dot(a.numpy(), b.numpy())

    def axpy(self, y, alpha, x):
        return self.torch.add(y, self.torch.mul(x, alpha))

    def axmy(self, y, alpha, x):
        return self.torch.sub(y, self.torch.mul(x, alpha))

    def take(self, v, idx):
        return v[self.torch.as_tensor(np.asarray(idx))]

    def sub(self, a, b):
        return self.torch.sub(a, b)


class SingleComm:
    rank, world = 0, 1

    def allreduce_(self, t):
        return t

    def allreduce_scalar(self, v):
        return v

    def allgather_cat(self, t, sizes):
        return t


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


def test_local_rows_products_sum_to_global():
    S, b, pre, cfg, na = problem()
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal(S.ncols), rng.standard_normal(S.nrows)
    parts = [D.local_rows(S, lo, hi) for lo, hi in D.row_blocks(S.nrows, 3)]
    assert np.array_equal(np.concatenate([O.matvec(P_, x) for P_ in parts]), O.matvec(S, x))
    zsum = sum(O.matvec_transpose(P_, y[lo:hi]) for P_, (lo, hi) in zip(parts, D.row_blocks(S.nrows, 3)))
    assert np.allclose(zsum, O.matvec_transpose(S, y), rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("mode", ["cg", "identity", "dense"])
def test_single_rank_is_bitwise_pcgls(mode):
    S, b, pre, cfg, na = problem(mode)
    x1, rep1 = D.pcgls_row_partitioned(S, b, pre, cfg, SingleComm(), CpuBackend)
    xo, repo = O.pcgls(S, b, O.OraclePreconditioner.from_reference(pre), na, delta=cfg.delta,
                       max_iters=cfg.max_iters)
    assert np.array_equal(x1, xo)
    assert rep1.its == repo["its"] and rep1.converged == repo["converged"]
    assert rep1.ratio_pt_history == repo["ratio_pt_history"]
    assert rep1.residual_norm_final == repo["residual_norm"]


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S, b, pre, cfg, na = problem()
        comm = D.TorchComm()
        x, rep = D.pcgls_row_partitioned(S, b, pre, cfg, comm, CpuBackend)
        if rank == 0:
            np.save(out, np.concatenate([[rep.its, rep.converged, rep.residual_norm_final], x]))
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_matches_single(tmp_path):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = str(tmp_path / "r0.npy")
    mp.start_processes(_worker, args=(2, port, out), nprocs=2, join=True, start_method="spawn")
    got = np.load(out)
    S, b, pre, cfg, na = problem()
    x1, rep1 = D.pcgls_row_partitioned(S, b, pre, cfg, SingleComm(), CpuBackend)
    assert int(got[0]) == rep1.its and bool(got[1]) == rep1.converged
    assert abs(got[2] - rep1.residual_norm_final) <= 1e-10 * rep1.residual_norm_final
    x2 = got[3:]
    assert np.linalg.norm(x2 - x1) <= 1e-10 * np.linalg.norm(x1)
