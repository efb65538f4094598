"""The C-ABI library loads and exports every symbol include/rowsplit_b200.h
declares; without a GPU the device entry points fail loudly (no CPU
fallback), while the host-setup entry points work."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "rowsplit_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(rsb_[a-z0-9_]+)\s*\(", text)))


def test_header_symbols_exported():
    from paper_2603_28642_b200 import _lib

    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 40
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) <= set(_lib.exported_symbols()) | {"rsb_last_error"}


def test_no_cpu_fallback_without_device():
    from paper_2603_28642_b200 import _lib as L

    c = ctypes.c_int(-1)
    L.check(L.lib().rsb_device_count(ctypes.byref(c)))
    if c.value > 0:
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    rc = L.lib().rsb_ctx_create(0, 0, ctypes.byref(h))
    assert rc == L.RSB_ECUDA
    assert b"no CUDA device" in L.lib().rsb_last_error()
    import paper_2603_28642_b200 as P

    with pytest.raises(RuntimeError):
        P.matvec(P.CscMatrix.identity(2), np.ones(2))


def test_api_surface_mirrors_reference():
    import paper_2603_28642_b200 as P

    for name in ["CglsConfig", "CscMatrix", "DenseMatrix", "IlupFactors", "IlupParams", "Permutation",
                 "RowSplitPreconditioner", "SMode", "SolveReport", "YMode", "build_preconditioner",
                 "build_y_explicit", "assemble_s_dense", "column_scale", "dense_cholesky_factorize",
                 "dense_cholesky_solve", "error_estimate", "ilup_factorize", "matvec", "matvec_transpose",
                 "pcgls", "power_method_norm2", "sparse_lower_solve", "sparse_lower_solve_transpose",
                 "sparse_upper_solve", "sparse_upper_solve_transpose", "stopping_ratio"]:
        assert hasattr(P, name), name
    assert P.error_estimate([(2.0, 3.0)], 1) == 6.0
    assert P.error_estimate([(1.0, 1.0), (2.0, 2.0), (3.0, 3.0)], 2) == 13.0
    assert P.stopping_ratio(1e-20, 1.0, 0.0, 1.0) == pytest.approx(1e-10)
    with pytest.raises(ValueError):
        P.stopping_ratio(1.0, 0.0, 0.0, 0.0)
    with pytest.raises(ValueError):
        P.CglsConfig(norm_A=1.0, estimator_delay=0)
