"""Pin the oracle (oracle/) to the reference before trusting it.

Every fixture under tests/golden/ was produced by the reference package
itself (tests/golden/make_golden.py); the oracle must reproduce all of it
bit for bit.  When the reference is importable (build container) the same
checks also run live against it on fresh seeds.
"""

import os

import numpy as np
import pytest

from conftest import csc_from, factors_from, golden, golden_json, reference
from oracle import oracle as O


@pytest.fixture(scope="module")
def K():
    return golden("kernels.npz")


def test_oracle_spmv_bitwise(K):
    c = 0
    while f"mv{c}_shape" in K:
        A = csc_from(K, f"mv{c}")
        assert np.array_equal(O.matvec(A, K[f"mv{c}_x"]), K[f"mv{c}_Ax"]), c
        assert np.array_equal(O.matvec_transpose(A, K[f"mv{c}_y"]), K[f"mv{c}_ATy"]), c
        c += 1
    assert c >= 5


def test_oracle_triangular_bitwise(K):
    c = 0
    while f"tl{c}_shape" in K:
        Ls, Ln, U = csc_from(K, f"tl{c}"), csc_from(K, f"tn{c}"), csc_from(K, f"tu{c}")
        b = K[f"t{c}_b"]
        assert np.array_equal(O.sparse_lower_solve(Ls, b, unit_diag=True), K[f"t{c}_lower_unit"])
        assert np.array_equal(O.sparse_lower_solve(Ln, b), K[f"t{c}_lower"])
        assert np.array_equal(O.sparse_upper_solve(U, b), K[f"t{c}_upper"])
        assert np.array_equal(O.sparse_lower_solve_transpose(Ls, b, unit_diag=True), K[f"t{c}_lower_t_unit"])
        assert np.array_equal(O.sparse_lower_solve_transpose(Ln, b), K[f"t{c}_lower_t"])
        assert np.array_equal(O.sparse_upper_solve_transpose(U, b), K[f"t{c}_upper_t"])
        c += 1
    assert c >= 3


def test_oracle_cholesky_bitwise(K):
    c = 0
    while f"ch{c}_S" in K:
        G = O.dense_cholesky_factorize(K[f"ch{c}_S"])
        assert np.array_equal(G, K[f"ch{c}_G"])
        assert np.array_equal(O.dense_cholesky_solve(G, K[f"ch{c}_b"]), K[f"ch{c}_x"])
        c += 1


def test_oracle_blas_dot_order(K):
    """rso_blas_dot restates OpenBLAS ddot's association (SkylakeX, 1 thread)."""
    drng = np.random.default_rng(77)
    for n, want in zip(K["dot_lens"], K["dot_vals"]):
        a, b = drng.standard_normal(int(n)), drng.standard_normal(int(n))
        assert O.dot(a, b) == want, n


def test_oracle_pairwise_reduceat(K):
    seg, starts = K["pw_seg"], K["pw_starts"]
    ends = list(starts[1:]) + [len(seg)]
    for s, e, want in zip(starts, ends, K["pw_sums"]):
        got = seg[s] + O.pairwise_sum(seg[s + 1:e])
        assert got == want


def _oracle_matches_fixture(name, pm_seed):
    z = golden(f"{name}.npz")
    meta = golden_json(f"{name}_reports.json")
    S = csc_from(z, "S")
    f = factors_from(z)
    b, norm_a = z["b"], float(z["norm_a"])
    assert O.power_method_norm2(S, 100, pm_seed) == norm_a
    for mode, want in meta["reports"].items():
        if mode == "plain":
            x, rep = O.pcgls(S, b, None, norm_a, delta=meta["delta"], max_iters=meta["max_iters"])
        else:
            Y = csc_from(z, f"Y_{mode}") if f"Y_{mode}_shape" in z else None
            G = z[f"G_{mode}"] if f"G_{mode}" in z else None
            pre = O.OraclePreconditioner(f, mode, "explicit" if mode == "dense" else "implicit", 2, Y, G,
                                         want["psize"])
            assert np.array_equal(pre.apply(z["r1"], z["r2"]), z[f"h_{mode}"]), mode
            assert np.array_equal(pre.y_apply(z["r1"]), z[f"yapply_{mode}"]), mode
            assert np.array_equal(pre.y_apply_transpose(z["r2"]), z[f"yapplyT_{mode}"]), mode
            assert np.array_equal(pre.s_matvec_implicit(z["r2"]), z[f"smv_{mode}"]), mode
            x, rep = O.pcgls(S, b, pre, norm_a, delta=meta["delta"], max_iters=meta["max_iters"])
        assert np.array_equal(x, z[f"x_{mode}"]), mode
        assert rep == want, mode


@pytest.mark.parametrize("name", ["cfg0s_mu0.1", "cfg0s_mu1.0", "cfg1s_mu1.0"])
def test_oracle_apply_and_pcgls_bitwise(name):
    _oracle_matches_fixture(name, 0)


@pytest.fixture
def blas_threads():
    prev = O.set_blas_threads(1)
    yield O.set_blas_threads
    O.set_blas_threads(prev)


def test_oracle_blas_threads_split():
    """OpenBLAS's thread split (blas_l1_thread.c): one thread up to 10000."""
    assert O.blas_chunks(10000, 8) == [10000]
    assert O.blas_chunks(10001, 8) == [1251, 1250, 1250, 1250, 1250, 1250, 1250, 1250]
    assert O.blas_chunks(20001, 3) == [6667, 6667, 6667]
    assert sum(O.blas_chunks(1000003, 64)) == 1000003


def test_oracle_blas_threads_dot_order(blas_threads):
    """The reference's numpy at OPENBLAS_NUM_THREADS = 2, 4, 8 (dots_mt.json,
    tests/golden/make_golden_mt.py)."""
    g = golden_json("dots_mt.json")
    for t, vals in g["dots"].items():
        blas_threads(int(t))
        rng = np.random.default_rng(g["seed"])
        for n, want in zip(g["lens"], vals):
            a, b = rng.standard_normal(n), rng.standard_normal(n)
            assert O.dot(a, b) == want, (t, n)


def test_oracle_pcgls_blas_threads_golden(blas_threads):
    """The whole reference pipeline run with OPENBLAS_NUM_THREADS=8 on a
    112^2-grid config 1 (every n- and m-long dot and norm threaded)."""
    blas_threads(8)
    _oracle_matches_fixture("cfg1m_t8", 1)


def test_oracle_identity_golden():
    """The reference's golden_identity case: history [1.0, 0.0] pins the
    stopped-early partial-window branch (sv.py:235-253)."""
    from paper_2603_28642_b200.types import CscMatrix, Permutation
    from paper_2603_28642_b200.ilup import IlupFactors

    g = golden_json("identity5.json")
    A = CscMatrix.identity(5)
    f = IlupFactors(Permutation.identity(5), CscMatrix.from_coo(5, 5, [], [], []),
                    CscMatrix.from_coo(0, 5, [], [], []), CscMatrix.identity(5), 0, np.zeros(5, np.int64))
    pre = O.OraclePreconditioner(f, "dense", "explicit", 2, CscMatrix.from_coo(0, 5, [], [], []),
                                 np.zeros((0, 0)), 5)
    x, rep = O.pcgls(A, np.array(g["b"]), pre, g["norm_a"], delta=1e-10)
    assert rep == g["report"]
    assert rep["ratio_pt_history"] == [1.0, 0.0]
    assert x.tolist() == g["x"]


def test_oracle_live_against_reference():
    """Fresh seeds, the live reference (skipped on the GPU box)."""
    rs = reference()
    if os.environ.get("OPENBLAS_NUM_THREADS") not in ("1", None):
        pytest.skip("long BLAS dots are thread-count dependent in the reference")
    rng = np.random.default_rng(4242)
    for _ in range(20):
        m, n = int(rng.integers(2, 90)), int(rng.integers(1, 70))
        a = rng.standard_normal((m, n)) * (rng.random((m, n)) < rng.uniform(0.05, 0.9))
        A = rs.CscMatrix.from_dense(a)
        x, y = rng.standard_normal(n), rng.standard_normal(m)
        assert np.array_equal(O.matvec(A, x), rs.matvec(A, x))
        assert np.array_equal(O.matvec_transpose(A, y), rs.matvec_transpose(A, y))
        k = min(m, n)
        low = rs.CscMatrix.from_dense(np.tril(a[:k, :k], -1))
        b = rng.standard_normal(k)
        assert np.array_equal(O.sparse_lower_solve(low, b, True), rs.sparse_lower_solve(low, b, True))
        assert np.array_equal(O.sparse_lower_solve_transpose(low, b, True),
                              rs.sparse_lower_solve_transpose(low, b, True))
