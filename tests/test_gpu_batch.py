"""The batched solve (csrc/bsolver.cu): up to 8 right-hand sides through
kernels that read each matrix and factor entry once for all of them.

SURVEY.md 8(e): config 4's 64 RHS run 8 per GPU with replicated factors.
The reference solves one b per pcgls call (sv.py:120-126), so the bar is:
every RHS of a batch gives the x and SolveReport of its own single pcgls,
bit for bit -- including RHS that stop at different iterations, a zero RHS
(the z.z == 0 start) and partial batches.
"""

import json
import os

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from oracle import oracle as O
from paper_2603_28642_b200 import device as D
from paper_2603_28642_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _rep(r):
    return json.dumps(r.to_dict() if hasattr(r, "to_dict") else r, sort_keys=True)


@pytest.fixture(scope="module")
def cfg4():
    """configs[4] structure at n = 200,000, mu = 1: wide DAGs (grid schedules)."""
    A, B = W.config4(seed=4, n=200_000, nrhs=11)
    S, _ = P.column_scale(A)
    na = P.power_method_norm2(S, 100, 4)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=0.0, mu=1.0))
    return S, B, na, f


def _singles(S, B, pre, cfg):
    out = []
    for j in range(B.shape[0]):
        out.append(P.pcgls(S, B[j], pre, cfg))
    return out


@pytest.mark.parametrize("mode", ["cg", "identity"])
def test_batch_equals_single_solves(cfg4, mode):
    S, B, na, f = cfg4
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
    dA = D.device_matrix(S)
    assert D.device_batch_solver(dA, D.device_preconditioner(pre, dA.ctx)) is not None, "batched path not taken"
    # a realistic tolerance: the RHS certify at different iterations
    cfg = P.CglsConfig(norm_A=na, delta=1e-8, max_iters=60)
    Bm = B[:8].copy()
    Bm[5] = 0.0  # z.z == 0 at the start (sv.py:184-196)
    X, reps = P.pcgls_batch(S, Bm, pre, cfg)
    singles = _singles(S, Bm, pre, cfg)
    its = set()
    for j, (x1, r1) in enumerate(singles):
        assert np.array_equal(X[j], x1, equal_nan=True), f"rhs {j}: iterate differs"
        assert _rep(reps[j]) == _rep(r1), f"rhs {j}: report differs"
        its.add(r1.its)
    assert len(its) > 1, "every RHS stopped at the same iteration; the per-RHS control is not exercised"


def test_batch_fixed_iterations_partial_and_multi(cfg4):
    """delta = 1e-300 (the bench protocol) with 3 RHS (a partial batch) and
    with 11 RHS (a full batch plus a partial one); one RHS checked against
    the oracle as well."""
    S, B, na, f = cfg4
    pre = P.build_preconditioner(f, s_mode=P.SMode.INNER_CG)
    cfg = P.CglsConfig(norm_A=na, delta=1e-300, max_iters=7)
    for k in (3, 11):
        X, reps = P.pcgls_batch(S, B[:k], pre, cfg)
        for j, (x1, r1) in enumerate(_singles(S, B[:k], pre, cfg)):
            assert np.array_equal(X[j], x1), (k, j)
            assert _rep(reps[j]) == _rep(r1), (k, j)
    op = O.OraclePreconditioner.from_reference(pre)
    xo, ro = O.pcgls(S, B[2], op, na, delta=1e-300, max_iters=7)
    assert np.array_equal(X[2], xo)
    ro["psize"] = pre.psize
    assert _rep(reps[2]) == _rep(ro)


def test_batch_plain_cgls(cfg4):
    """pre = None (plain CGLS, h = A^T r) through the batched kernels."""
    S, B, na, _ = cfg4
    cfg = P.CglsConfig(norm_A=na, delta=1e-6, max_iters=40)
    X, reps = P.pcgls_batch(S, B[:4], None, cfg)
    for j, (x1, r1) in enumerate(_singles(S, B[:4], None, cfg)):
        assert np.array_equal(X[j], x1), j
        assert _rep(reps[j]) == _rep(r1), j


def test_batch_streams_path_still_available(cfg4, monkeypatch):
    """RSB_BATCH=streams keeps the one-stream-per-RHS path (same results)."""
    S, B, na, f = cfg4
    pre = P.build_preconditioner(f, s_mode=P.SMode.IDENTITY)
    cfg = P.CglsConfig(norm_A=na, delta=1e-300, max_iters=4)
    Xb, rb = P.pcgls_batch(S, B[:2], pre, cfg)
    monkeypatch.setenv("RSB_BATCH", "streams")
    Xs, rs_ = P.pcgls_batch(S, B[:2], pre, cfg)
    assert np.array_equal(Xb, Xs) and [_rep(r) for r in rb] == [_rep(r) for r in rs_]


def test_batch_rejects_narrow_and_dense():
    """Narrow DAGs (single-CTA solves) and the dense coupling stay on the
    stream path: the batched solver declines them."""
    A, b = W.config0(seed=0, m=600, n=400)
    S, _ = P.column_scale(A)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=1e-3, mu=1.0))
    for mode in (P.SMode.DENSE_FACTOR, P.SMode.INNER_CG):
        pre = P.build_preconditioner(f, s_mode=mode)
        dA = D.device_matrix(S)
        assert D.device_batch_solver(dA, D.device_preconditioner(pre, dA.ctx)) is None
        X, reps = P.pcgls_batch(S, np.stack([b, b]), pre, P.CglsConfig(norm_A=1.0, delta=1e-8, max_iters=20))
        x1, r1 = P.pcgls(S, b, pre, P.CglsConfig(norm_A=1.0, delta=1e-8, max_iters=20))
        assert np.array_equal(X[1], x1) and _rep(reps[1]) == _rep(r1)


def test_batch_static_schedule_option(cfg4, monkeypatch):
    """RSB_TRSV_GRID=static: the batched static-schedule solve (opt-in) gives
    the same bits."""
    S, B, na, f = cfg4
    pre = P.build_preconditioner(f, s_mode=P.SMode.INNER_CG)
    cfg = P.CglsConfig(norm_A=na, delta=1e-300, max_iters=5)
    X0, r0 = P.pcgls_batch(S, B[:8], pre, cfg)
    monkeypatch.setenv("RSB_TRSV_GRID", "static")
    D.clear_caches()
    A2 = P.CscMatrix(S.nrows, S.ncols, S.col_ptr, S.row_idx, S.values)
    pre2 = P.build_preconditioner(f, s_mode=P.SMode.INNER_CG)
    X1, r1 = P.pcgls_batch(A2, B[:8], pre2, cfg)
    assert np.array_equal(X0, X1) and [_rep(r) for r in r0] == [_rep(r) for r in r1]


@pytest.mark.parametrize("mode", ["cg", "identity"])
def test_batch_index_order_solve(cfg4, mode, monkeypatch):
    """RSB_TRSV_ORDER=natural + RSB_BTRSV_NAT=1: the index-order batched solve
    (btrsv_nat.cu, opt-in) against the single solves
    through the level-ordered kernels, incl. a zero RHS and different stop
    iterations."""
    S, B, na, f = cfg4
    cfg = P.CglsConfig(norm_A=na, delta=1e-8, max_iters=60)
    Bm = B[:8].copy()
    Bm[5] = 0.0
    monkeypatch.setenv("RSB_TRSV_ORDER", "level")
    D.clear_caches()
    pre0 = P.build_preconditioner(f, s_mode=P.SMode(mode))
    singles = _singles(S, Bm, pre0, cfg)
    monkeypatch.setenv("RSB_TRSV_ORDER", "natural")
    monkeypatch.setenv("RSB_BTRSV_NAT", "1")
    D.clear_caches()
    A2 = P.CscMatrix(S.nrows, S.ncols, S.col_ptr, S.row_idx, S.values)
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
    from paper_2603_28642_b200 import _lib as L

    dpre = D.device_preconditioner(pre, D.get_context())
    assert dpre.L1.variant(L.TRI_LOWER_UNIT)[0] == "natural" and dpre.U.variant(L.TRI_UPPER)[0] == "natural"
    X, reps = P.pcgls_batch(A2, Bm, pre, cfg)
    for j, (x1, r1) in enumerate(singles):
        assert np.array_equal(X[j], x1, equal_nan=True), f"rhs {j}: iterate differs"
        assert _rep(reps[j]) == _rep(r1), f"rhs {j}: report differs"
    D.clear_caches()
