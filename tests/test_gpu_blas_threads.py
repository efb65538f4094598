"""The device's RSB_BLAS_THREADS=T dot order vs the reference run with
OPENBLAS_NUM_THREADS=T.

numpy's OpenBLAS splits every dot longer than 10000 over T threads (T
contiguous chunks, partial results summed in chunk order).  With
RSB_BLAS_THREADS=T the device reproduces that split: one block per chunk,
each the one-thread association, the last block combining.  Pinned against
the reference's own multi-threaded outputs (tests/golden/make_golden_mt.py)
and against the oracle at T up to 64, including chunks that start on odd
elements (the bulk copies' alignment shift) and vectors of odd length.
"""

import json

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from conftest import csc_from, factors_from, golden, golden_json
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture
def threads(monkeypatch):
    prev = O.set_blas_threads(1)

    def use(t):
        monkeypatch.setenv("RSB_BLAS_THREADS", str(t))
        O.set_blas_threads(t)

    yield use
    O.set_blas_threads(prev)


def _device_dot(a, b):
    from paper_2603_28642_b200 import _lib as L
    from paper_2603_28642_b200.device import get_context

    out = np.zeros(1)
    L.check(L.lib().rsb_dot(get_context().h, len(a), L.ptr(a), L.ptr(b), out.ctypes.data_as(L.f64p), L.RSB_HOST))
    return out[0]


def test_reference_multithread_dots(threads):
    g = golden_json("dots_mt.json")
    for t, vals in g["dots"].items():
        threads(int(t))
        rng = np.random.default_rng(g["seed"])
        for n, want in zip(g["lens"], vals):
            a, b = rng.standard_normal(n), rng.standard_normal(n)
            assert _device_dot(a, b) == want, (t, n)


def test_b200_host_multithread_dots(threads):
    """The device's T-thread dot order against numpy run on the B200 box's own
    16-core host at T = 12 and 16 (tests/golden/dots_mt_host.json), incl. the
    config-4 lengths 8e6 and 1.6e7."""
    g = golden_json("dots_mt_host.json")
    for t in ("12", "16"):
        threads(int(t))
        rng = np.random.default_rng(g["seed"])
        for n, want in zip(g["lens"], g["dots"][t]):
            a, b = rng.standard_normal(n), rng.standard_normal(n)
            assert _device_dot(a, b) == want, (t, n)


@pytest.mark.parametrize("t", [2, 3, 7, 16, 33, 64])
@pytest.mark.parametrize("n", [10000, 10001, 98304, 24577 * 7, 1_000_003, 1_500_000, 4_000_001])
def test_device_dot_threads_vs_oracle(threads, t, n):
    threads(t)
    rng = np.random.default_rng(n + t)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    assert _device_dot(a, b) == O.dot(a, b)


def test_pcgls_reference_multithread_golden(threads):
    """configs[1] at a 112^2 grid, the reference pipeline at
    OPENBLAS_NUM_THREADS=8: power method, apply and pcgls bit for bit."""
    threads(8)
    z = golden("cfg1m_t8.npz")
    meta = golden_json("cfg1m_t8_reports.json")
    S = csc_from(z, "S")
    f = factors_from(z)
    b, norm_a = z["b"], float(z["norm_a"])
    assert P.power_method_norm2(S, 100, 1) == norm_a
    cfg = P.CglsConfig(norm_A=norm_a, delta=meta["delta"], max_iters=meta["max_iters"])
    for mode, want in meta["reports"].items():
        pre = None if mode == "plain" else P.build_preconditioner(f, s_mode=P.SMode(mode))
        if pre is not None:
            assert np.array_equal(pre.apply(z["r1"], z["r2"]), z[f"h_{mode}"]), mode
        x, rep = P.pcgls(S, b, pre, cfg)
        assert np.array_equal(x, z[f"x_{mode}"]), mode
        assert rep.to_dict() == want, mode


@pytest.mark.parametrize("t", [8, 64])
def test_pcgls_threads_config4_structure_vs_oracle(threads, t):
    """configs[4] structure at n = 60,000 (n-, m- and s-long dots all
    threaded), cg(2) and identity, fixed 8 iterations plus the batch path."""
    from paper_2603_28642_b200 import workloads as W

    threads(t)
    A, B = W.config4(seed=4, n=60_000, nrhs=2)
    S, _ = P.column_scale(A)
    na = P.power_method_norm2(S, 100, 4)
    assert na == O.power_method_norm2(S, 100, 4)
    f = P.ilup_factorize(S, P.IlupParams(p=10, tau=0.0, mu=1.0))
    for mode in ("cg", "identity"):
        pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
        op = O.OraclePreconditioner.from_reference(pre)
        cfg = P.CglsConfig(norm_A=na, delta=1e-300, max_iters=8)
        X, reps = P.pcgls_batch(S, B, pre, cfg)
        for j in range(2):
            xo, repo = O.pcgls(S, B[j], op, na, delta=1e-300, max_iters=8)
            assert np.array_equal(X[j], xo), (mode, j)
            assert json.dumps(reps[j].to_dict(), sort_keys=True) == json.dumps(repo, sort_keys=True)
