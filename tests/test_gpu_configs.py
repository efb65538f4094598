"""Device pcgls vs the oracle on every BASELINE.json configuration.

Each config's generator (paper_2603_28642_b200/workloads.py) at a size the
single-thread oracle finishes in seconds, through the reference pipeline
order (cli.py:59-94): column_scale (not config 3), power_method_norm2,
ilup_factorize, build_preconditioner, pcgls -- every coupling mode the
config runs.  The bar is bit-identity: x, the whole
SolveReport (its, flags, ratio history, final norms) and one
preconditioner application.  Config 1 also runs at its full BASELINE size.
"""

import json

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from oracle import oracle as O
from paper_2603_28642_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _pipeline(A, scale, mu, tau, seed):
    S = P.column_scale(A)[0] if scale else A
    na = P.power_method_norm2(S, 100, seed)
    assert na == O.power_method_norm2(S, 100, seed)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=tau, mu=mu))
    return S, na, f


def _same_report(got, want):
    # json text compares NaN entries of the ratio history as equal
    return json.dumps(got.to_dict(), sort_keys=True) == json.dumps(want, sort_keys=True)


def _check(S, b, na, f, mode, delta, max_iters, seed, fixed=0):
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
    op = O.OraclePreconditioner.from_reference(pre)
    # one application on identical inputs (the north star's 1e-10 bar; here bitwise)
    rng = np.random.default_rng(seed)
    n = S.ncols
    r1, r2 = rng.standard_normal(n), rng.standard_normal(S.nrows - n)
    h = pre.apply(r1, r2)
    ho = op.apply(r1, r2)
    assert np.array_equal(h, ho, equal_nan=True), f"{mode}: apply differs"
    x, rep = P.pcgls(S, b, pre, P.CglsConfig(norm_A=na, delta=delta, max_iters=max_iters))
    xo, repo = O.pcgls(S, b, op, na, delta=delta, max_iters=max_iters)
    assert np.array_equal(x, xo, equal_nan=True), f"{mode}: iterate differs"
    assert _same_report(rep, repo), f"{mode}: report differs"
    if fixed:
        # the throughput protocol: exactly `fixed` iterations (delta = 1e-300)
        x, rep2 = P.pcgls(S, b, pre, P.CglsConfig(norm_A=na, delta=1e-300, max_iters=fixed))
        xo, repo = O.pcgls(S, b, op, na, delta=1e-300, max_iters=fixed)
        assert np.array_equal(x, xo, equal_nan=True), f"{mode}: fixed-iteration iterate differs"
        assert _same_report(rep2, repo), f"{mode}: fixed-iteration report differs"
    return rep


@pytest.mark.parametrize("mode", ["cg", "identity"])
def test_config1_full_size(mode):
    """configs[1] at its BASELINE size (n = 65,536, m = 98,304), mu = 1."""
    A, b = W.config1(seed=1)
    S, na, f = _pipeline(A, True, 1.0, 0.0, 1)
    rep = _check(S, b, na, f, mode, 1e-10, 40, 1)
    assert rep.its > 0


@pytest.mark.parametrize("mu", [0.1, 1.0])
@pytest.mark.parametrize("mode", ["dense", "cg", "identity"])
def test_config2_dense_rows(mu, mode):
    """configs[2] structure (6 nnz/row + 100 rows with 50% of columns) at
    n = 6,000: the dense rows land in the s = 100 coupling system (the
    Woodbury/Cholesky path in dense mode)."""
    A, b = W.config2(seed=2, n=6000)
    S, na, f = _pipeline(A, True, mu, 0.0, 2)
    assert f.L2.nrows == 100
    _check(S, b, na, f, mode, 1e-8, 150, 2, fixed=25)


@pytest.mark.parametrize("mu", [0.1, 1.0])
@pytest.mark.parametrize("mode", ["cg", "identity"])
def test_config3_ill_conditioned_unscaled(mu, mode):
    """configs[3] structure (8 nnz/row, column scales 10^U(-4,4), run
    unscaled) at n = 3,000."""
    A, b = W.config3(seed=3, n=3000)
    S, na, f = _pipeline(A, False, mu, 0.0, 3)
    _check(S, b, na, f, mode, 1e-8, 150, 3, fixed=25)


@pytest.mark.parametrize("mode", ["cg", "identity"])
def test_config4_structure_batch(mode):
    """configs[4] structure (6 nnz/row, m = 2n, mu = 1) at n = 20,000: four
    right-hand sides from the config's RHS stream solved concurrently by
    pcgls_batch, each bit-identical to the oracle's single solve."""
    A, B = W.config4(seed=4, n=20_000, nrhs=4)
    S, na, f = _pipeline(A, True, 1.0, 0.0, 4)
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
    op = O.OraclePreconditioner.from_reference(pre)
    cfg = P.CglsConfig(norm_A=na, delta=1e-8, max_iters=80)
    X, reports = P.pcgls_batch(S, B, pre, cfg)
    assert X.shape == (4, S.ncols) and len(reports) == 4
    for j in range(4):
        xo, repo = O.pcgls(S, B[j], op, na, delta=1e-8, max_iters=80)
        assert np.array_equal(X[j], xo), f"rhs {j}: iterate differs"
        assert _same_report(reports[j], repo), f"rhs {j}: report differs"


@pytest.mark.parametrize("order", ["natural", "level"])
def test_config4_structure_solve_order(order, monkeypatch):
    """The same structure with the wide solves forced to the index-order
    kernel (trsv_nat.cu; the default at n = 8e6, where dependencies are far)
    and to the level-ordered one: both bit-identical to the oracle."""
    from paper_2603_28642_b200 import _lib as L
    from paper_2603_28642_b200 import device

    monkeypatch.setenv("RSB_TRSV_ORDER", order)
    device.clear_caches()
    A, B = W.config4(seed=4, n=200_000, nrhs=1)
    S, na, f = _pipeline(A, True, 1.0, 0.0, 4)
    want = "natural" if order == "natural" else "grid"
    for M, kind in ((f.L1, L.TRI_LOWER_UNIT), (f.L1, L.TRI_LOWER_T_UNIT), (f.U, L.TRI_UPPER)):
        Mc = P.CscMatrix(M.nrows, M.ncols, M.col_ptr, M.row_idx, M.values)
        assert device.DeviceMatrix(Mc, device.get_context()).variant(kind)[0] == want
    _check(S, B[0], na, f, "cg", 1e-300, 6, 4)
    device.clear_caches()


def test_config4_structure_fixed_iterations_wide_dag():
    """configs[4] structure at n = 200,000 (wide DAGs: the grid-wide
    sync-free solve) for a fixed 6 iterations (delta = 1e-300, the bench's
    throughput protocol): iterate and report bit-identical to the oracle."""
    A, B = W.config4(seed=4, n=200_000, nrhs=1)
    S, na, f = _pipeline(A, True, 1.0, 0.0, 4)
    _check(S, B[0], na, f, "cg", 1e-300, 6, 4)


@pytest.mark.parametrize("cg_iters", [1, 2, 3])
def test_index_order_solve_chain_across_solves(cg_iters, monkeypatch):
    """The index-order solves of one application fill each other's outputs
    with the sentinel (TrsvChain, csrc/solver.cu), the last one refilling the
    next application's first output.  One solver runs to convergence (its
    gated tail must leave the chain intact), stops at max_iters, and is
    started again with other right-hand sides, with standalone applications
    (the preconditioner's own workspace) in between: all bit-identical to the
    oracle, for 1 / 2 / 3 inner CG steps (odd steps use the second buffer)."""
    from paper_2603_28642_b200 import device

    monkeypatch.setenv("RSB_TRSV_ORDER", "natural")
    device.clear_caches()
    A, B = W.config4(seed=14, n=100_000, nrhs=3)
    S, na, f = _pipeline(A, True, 1.0, 0.0, 14)
    pre = P.build_preconditioner(f, s_mode=P.SMode("cg"), cg_iters=cg_iters)
    op = O.OraclePreconditioner.from_reference(pre)
    rng = np.random.default_rng(99)
    n = S.ncols
    for j, (delta, its) in enumerate(((1e-8, 60), (1e-300, 4), (1e-6, 60))):
        x, rep = P.pcgls(S, B[j], pre, P.CglsConfig(norm_A=na, delta=delta, max_iters=its))
        xo, repo = O.pcgls(S, B[j], op, na, delta=delta, max_iters=its)
        assert np.array_equal(x, xo, equal_nan=True), f"solve {j}: iterate differs"
        assert _same_report(rep, repo), f"solve {j}: report differs"
        r1, r2 = rng.standard_normal(n), rng.standard_normal(S.nrows - n)
        assert np.array_equal(pre.apply(r1, r2), op.apply(r1, r2), equal_nan=True), f"apply after solve {j} differs"
    device.clear_caches()
