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


def test_oracle_blas_threads_dot_order_b200_host(blas_threads):
    """numpy on the B200 box's 16-core host at OPENBLAS_NUM_THREADS = 1 .. 16
    (dots_mt_host.json, written there by scripts/dot_probe_host.py
    --write-golden), up to the config-4 dot lengths 8e6 and 1.6e7."""
    g = golden_json("dots_mt_host.json")
    assert g["cores"] >= 16 and "16" in g["dots"]
    for t in ("12", "16"):
        blas_threads(int(t))
        rng = np.random.default_rng(g["seed"])
        for n, want in zip(g["lens"], g["dots"][t]):
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


# ---- host setup restatements and the threaded evaluation (bench.py's
# reference arm uses these instead of any product code)


def _same(a, b):
    return (a.nrows, a.ncols) == (b.nrows, b.ncols) and np.array_equal(a.col_ptr, b.col_ptr) \
        and np.array_equal(a.row_idx, b.row_idx) and np.array_equal(a.values, b.values)


@pytest.mark.parametrize("name", ["cfg0s_mu0.1", "cfg0s_mu1.0", "cfg1s_mu1.0"])
def test_oracle_setup_matches_reference_fixtures(name):
    from paper_2603_28642_b200 import workloads as W

    z = golden(f"{name}.npz")
    prm = golden_json(f"{name}_reports.json")["params"]
    A, _ = W.config0(seed=0, m=600, n=400) if name.startswith("cfg0") else W.config1(seed=1, g=24)
    S, scale = O.column_scale(A)
    assert _same(S, csc_from(z, "S")) and np.array_equal(scale, z["scale"])
    f = O.ilup_factorize(S, **prm)
    want = factors_from(z)
    assert np.array_equal(f.row_perm.perm, want.row_perm.perm)
    for k in ("L1", "L2", "U"):
        assert _same(getattr(f, k), getattr(want, k)), k
    assert f.nmod == want.nmod and np.array_equal(f.row_counts_final, want.row_counts_final)


def test_oracle_ilup_config4_n1e5_matches_reference_hashes():
    """Digests of the reference's own column_scale + ilup_factorize at the
    config-4 structure, n = 1e5, mu = 1 (tests/golden/make_cfg4_hashes.py)."""
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_cfg4_hashes import factor_digests

    from paper_2603_28642_b200 import workloads as W

    want = golden_json("cfg4_factor_hashes.json")["100000"]
    A, _ = W.config4(seed=4, n=100_000, nrhs=0)
    S, scale = O.column_scale(A)
    f = O.ilup_factorize(S, p=10, tau=0.0, mu=1.0)
    got = factor_digests(S.values, scale, f)
    for k, v in got.items():
        assert v == want[k], k


def test_oracle_ilup_random_vs_live_reference():
    rs = reference()
    rng = np.random.default_rng(5)
    for t in range(30):
        m = int(rng.integers(2, 60))
        n = int(rng.integers(1, m + 1))
        a = rng.standard_normal((m, n)) * (rng.random((m, n)) < rng.uniform(0.05, 1.0))
        if t % 4 == 0 and n > 2:
            a[:, 2 % n] = a[:, 0]
        for j in range(n):
            if not a[:, j].any():
                a[rng.integers(0, m), j] = 1.0
        prm = dict(p=int(rng.integers(1, 12)), tau=float(rng.choice([0.0, 1e-2, 0.3])),
                   mu=float(rng.choice([0.1, 0.5, 1.0])))
        A = rs.CscMatrix.from_dense(a)
        fr = rs.ilup_factorize(A, rs.IlupParams(**prm))
        fo = O.ilup_factorize(A, **prm)
        assert np.array_equal(fr.row_perm.perm, fo.row_perm.perm), t
        for k in ("L1", "L2", "U"):
            assert _same(getattr(fr, k), getattr(fo, k)), (t, k)
        assert fr.nmod == fo.nmod and np.array_equal(fr.row_counts_final, fo.row_counts_final)


def test_fast_kernels_match_sequential():
    """rsfast.c (threaded, level-scheduled, CSR) gives the sequential
    restatement's bits: kernels, the T-thread dot, a whole pcgls run."""
    from paper_2603_28642_b200 import workloads as W

    A, B = W.config4(seed=4, n=20_000, nrhs=1)
    S, _ = O.column_scale(A)
    f = O.ilup_factorize(S, p=10, tau=0.0, mu=1.0)
    rng = np.random.default_rng(3)
    x, y = rng.standard_normal(S.ncols), rng.standard_normal(S.nrows)
    prev_bt = O.set_blas_threads(8)
    try:
        seq = [O.matvec(S, x), O.matvec_transpose(S, y), O.sparse_lower_solve(f.L1, x, unit_diag=True),
               O.sparse_upper_solve(f.U, x), O.sparse_lower_solve_transpose(f.L1, x, unit_diag=True),
               O.dot(y, y), O.power_method_norm2(S, 5, 4)]
        pre = O.OraclePreconditioner(f, "cg", "implicit", 2)
        xs, rs_ = O.pcgls(S, B[0], pre, seq[-1], delta=1e-300, max_iters=4)
        prev = O.set_cpu_threads(4)
        try:
            fast = [O.matvec(S, x), O.matvec_transpose(S, y), O.sparse_lower_solve(f.L1, x, unit_diag=True),
                    O.sparse_upper_solve(f.U, x), O.sparse_lower_solve_transpose(f.L1, x, unit_diag=True),
                    O.dot(y, y), O.power_method_norm2(S, 5, 4)]
            xf, rf = O.pcgls(S, B[0], pre, seq[-1], delta=1e-300, max_iters=4)
        finally:
            O.set_cpu_threads(prev)
            O.clear_prep_cache()
    finally:
        O.set_blas_threads(prev_bt)
    for k, (a, b) in enumerate(zip(seq, fast)):
        assert np.array_equal(a, b), k
    assert np.array_equal(xs, xf) and rs_ == rf
