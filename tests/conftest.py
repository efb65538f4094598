import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN = os.path.join(REPO, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: full-size cases")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def golden_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def csc_from(z, prefix):
    from paper_2603_28642_b200.types import CscMatrix

    m, n = (int(v) for v in z[f"{prefix}_shape"])
    return CscMatrix(m, n, z[f"{prefix}_ptr"], z[f"{prefix}_idx"], z[f"{prefix}_val"])


def factors_from(z):
    from paper_2603_28642_b200.ilup import IlupFactors
    from paper_2603_28642_b200.types import Permutation

    return IlupFactors(Permutation.from_perm(z["perm"]), csc_from(z, "L1"), csc_from(z, "L2"),
                       csc_from(z, "U"), int(np.asarray(z["nmod"]).reshape(-1)[0]), z["row_counts"])


def reference():
    """The reference package, importable only in the build container."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference package not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import rowsplit

    return rowsplit


def rel_err(got, want):
    want = np.asarray(want, dtype=float)
    scale = np.linalg.norm(want)
    return np.linalg.norm(np.asarray(got) - want) / (scale if scale else 1.0)
