"""Device pcgls vs the oracle at the BASELINE.json sizes (configs 0, 1, 2).

Complements tests/test_gpu_configs.py (reduced sizes, every mode and mu):
here the configurations run at their stated sizes through the reference
pipeline order (cli.py:59-94) and the full solve to the config's tolerance
is compared bit for bit -- x, the whole SolveReport, one preconditioner
application.  The oracle runs its threaded, bit-identical kernels
(oracle/rsfast.c) so the checks finish in seconds.  Config 4 at n = 8e6 is
checked in every bench run (bench.py `parity`: x and report of a
fixed-iteration solve, factors against the reference's digests); config 3
at its full n needs hours of serial host ILUP and is checked at n = 1e5.
"""

import json
import os

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from oracle import oracle as O
from paper_2603_28642_b200 import workloads as W

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def oracle_threads():
    prev = O.set_cpu_threads(max(1, O.available_cores() - 1))
    yield
    O.set_cpu_threads(prev)
    O.clear_prep_cache()


def _same_report(got, want):
    return json.dumps(got.to_dict(), sort_keys=True) == json.dumps(want, sort_keys=True)


def _setup(A, scale, mu, tau, seed):
    S = P.column_scale(A)[0] if scale else A
    na = P.power_method_norm2(S, 100, seed)
    assert na == O.power_method_norm2(S, 100, seed)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=tau, mu=mu))
    return S, na, f


def _compare(S, b, na, f, mode, delta, max_iters, seed=0):
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
    op = O.OraclePreconditioner.from_reference(pre)
    rng = np.random.default_rng(seed)
    r1, r2 = rng.standard_normal(S.ncols), rng.standard_normal(S.nrows - S.ncols)
    assert np.array_equal(pre.apply(r1, r2), op.apply(r1, r2), equal_nan=True), f"{mode}: apply differs"
    x, rep = P.pcgls(S, b, pre, P.CglsConfig(norm_A=na, delta=delta, max_iters=max_iters))
    xo, repo = O.pcgls(S, b, op, na, delta=delta, max_iters=max_iters)
    assert np.array_equal(x, xo, equal_nan=True), f"{mode}: iterate differs"
    assert _same_report(rep, repo), f"{mode}: report differs"
    return rep


@pytest.mark.parametrize("mu", [0.1, 1.0])
@pytest.mark.parametrize("mode", ["dense", "cg", "identity"])
def test_config0_full_size(mu, mode):
    """configs[0]: m = 3000, n = 2000, tau = 1e-3, delta 1e-8, 2000 its."""
    A, b = W.config0(seed=0)
    S, na, f = _setup(A, True, mu, 1e-3, 0)
    _compare(S, b, na, f, mode, 1e-8, 2000)


def test_config1_full_size_to_tolerance():
    """configs[1] (n = 65,536, m = 98,304, mu = 1, cg(2)) solved to its
    delta = 1e-10 with the 2000-iteration cap: the whole run bitwise."""
    A, b = W.config1(seed=1)
    S, na, f = _setup(A, True, 1.0, 0.0, 1)
    rep = _compare(S, b, na, f, "cg", 1e-10, 2000)
    assert rep.its > 100


@pytest.fixture(scope="module")
def cfg2():
    A, b = W.config2(seed=2)  # n = 100,000, s = 100 dense rows
    S = P.column_scale(A)[0]
    na = P.power_method_norm2(S, 100, 2)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=0.0, mu=1.0))
    return S, b, na, f


@pytest.mark.parametrize("mode", ["dense", "cg", "identity"])
def test_config2_full_size(cfg2, mode):
    """configs[2] at n = 100,000 with its 100 dense rows (s = 100: the dense
    Woodbury/Cholesky coupling), mu = 1: a fixed 20-iteration run and the
    run to delta = 1e-8 (capped at 300 iterations), both bitwise."""
    S, b, na, f = cfg2
    assert f.L2.nrows == 100
    _compare(S, b, na, f, mode, 1e-300, 20, seed=2)
    _compare(S, b, na, f, mode, 1e-8, 300, seed=3)


def test_config3_structure_n1e5():
    """configs[3] structure (8 nnz/row, columns scaled by 10^U(-4,4), run
    unscaled) at n = 100,000, mu = 1, cg(2), delta 1e-8."""
    A, b = W.config3(seed=3, n=100_000)
    S, na, f = _setup(A, False, 1.0, 0.0, 3)
    _compare(S, b, na, f, "cg", 1e-8, 200)


def test_config2_dense_build_on_device(cfg2):
    """configs[2]'s dense coupling (s = 100 rows of Y over n = 100,000)
    built on the device: Y bit-identical to the host build
    (pinned to the reference), S within 1e-13 of numpy's product, the
    factor bitwise given S, the apply within 1e-10, and the solve to
    delta = 1e-8 takes the same number of iterations."""
    from paper_2603_28642_b200.precond import _gram_plus_identity, dense_build_device

    S, b, na, f = cfg2
    host = P.build_preconditioner(f, s_mode=P.SMode.DENSE_FACTOR, setup="host")
    Y, Sd, F, sec = dense_build_device(f, what=2)
    assert np.array_equal(Y.col_ptr, host.Y.col_ptr) and np.array_equal(Y.row_idx, host.Y.row_idx)
    assert np.array_equal(Y.values, host.Y.values)
    S_np = _gram_plus_identity(host.Y).a
    assert np.max(np.abs(Sd.a - S_np)) / np.max(np.abs(S_np)) <= 1e-13
    assert np.array_equal(F.a, P.dense_cholesky_factorize(Sd, setup="host").a)
    dev = P.build_preconditioner(f, s_mode=P.SMode.DENSE_FACTOR, setup="device")
    rng = np.random.default_rng(5)
    r1, r2 = rng.standard_normal(S.ncols), rng.standard_normal(S.nrows - S.ncols)
    h, hh = dev.apply(r1, r2), host.apply(r1, r2)
    assert np.linalg.norm(h - hh) / np.linalg.norm(hh) <= 1e-10
    cfg = P.CglsConfig(norm_A=na, delta=1e-8, max_iters=300)
    _, rep_d = P.pcgls(S, b, dev, cfg)
    _, rep_h = P.pcgls(S, b, host, cfg)
    assert rep_d.its == rep_h.its and rep_d.converged == rep_h.converged
    print(f"config2 device build: Y {sec[0]:.3f} s, S {sec[1]:.3f} s, factor {sec[2]:.3f} s")
