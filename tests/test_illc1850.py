"""illc1850, the reference's bundled paper matrix (pkg/data/illc1850.mtx;
paper Table 3 row 19; acceptance band pkg/tests/test_acceptance.py:155-175).

tests/golden/make_illc1850.py ran the reference's own pipeline on it (dense,
cg(2) and identity coupling: its = 12 / 6 / 3, all "converged").  The CPU
tests pin the oracle and the native host setup to those outputs; the GPU
test runs the device solve on the same inputs and requires the reference's
x, SolveReport and one preconditioner application bit for bit.
"""

import json

import numpy as np
import pytest

import paper_2603_28642_b200 as P
from conftest import csc_from, factors_from, golden, golden_json
from oracle import oracle as O


@pytest.fixture(scope="module")
def fx():
    return golden("illc1850.npz"), golden_json("illc1850.json")


def _same(a, b):
    return (a.nrows, a.ncols) == (b.nrows, b.ncols) and np.array_equal(a.col_ptr, b.col_ptr) \
        and np.array_equal(a.row_idx, b.row_idx) and np.array_equal(a.values, b.values)


def test_reference_counts_recorded(fx):
    _, meta = fx
    assert {m: r["its"] for m, r in meta["reports"].items()} == {"dense": 12, "cg": 6, "identity": 3}
    assert all(r["converged"] for r in meta["reports"].values())


def test_host_setup_reproduces_reference_factors(fx):
    """Oracle ILUP and the native ILUP both give the reference's factors."""
    z, meta = fx
    S = csc_from(z, "S")
    want = factors_from(z)
    for f in (O.ilup_factorize(S, **meta["params"]), P.ilup_factorize(S, P.IlupParams(**meta["params"]))):
        assert np.array_equal(f.row_perm.perm, want.row_perm.perm)
        for k in ("L1", "L2", "U"):
            assert _same(getattr(f, k), getattr(want, k)), k
        assert f.nmod == want.nmod
    assert O.power_method_norm2(S, 100, 42) == float(z["norm_A"][0])


@pytest.mark.parametrize("mode", ["dense", "cg", "identity"])
def test_oracle_reproduces_reference_solves(fx, mode):
    z, meta = fx
    S, f = csc_from(z, "S"), factors_from(z)
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode))  # host setup: Y and the S factor (pinned elsewhere)
    op = O.OraclePreconditioner.from_reference(pre)
    assert np.array_equal(op.apply(z["r1"], z["r2"]), z[f"h_{mode}"])
    x, rep = O.pcgls(S, z["b"], op, float(z["norm_A"][0]), delta=meta["delta"], max_iters=meta["max_iters"])
    assert np.array_equal(x, z[f"x_{mode}"])
    assert json.dumps(rep, sort_keys=True) == json.dumps(meta["reports"][mode], sort_keys=True)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["dense", "cg", "identity"])
def test_device_solve_matches_reference(fx, mode):
    z, meta = fx
    S, f = csc_from(z, "S"), factors_from(z)
    na = P.power_method_norm2(S, 100, 42)
    assert na == float(z["norm_A"][0])
    pre = P.build_preconditioner(f, s_mode=P.SMode(mode))
    assert np.array_equal(pre.apply(z["r1"], z["r2"]), z[f"h_{mode}"]), "apply differs from the reference"
    x, rep = P.pcgls(S, z["b"], pre, P.CglsConfig(norm_A=na, delta=meta["delta"], max_iters=meta["max_iters"]))
    assert np.array_equal(x, z[f"x_{mode}"]), "iterate differs from the reference"
    assert json.dumps(rep.to_dict(), sort_keys=True) == json.dumps(meta["reports"][mode], sort_keys=True)
