import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 and the built extension")
    config.addinivalue_line("markers", "slow: long-running parity case")


def load_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def golden_runs():
    return load_json("reference_runs.json")["runs"]


@pytest.fixture(scope="session")
def golden_assembly():
    return load_json("assembly_sha256.json")["matrices"]


@pytest.fixture(scope="session")
def spmv_cases():
    with np.load(os.path.join(GOLDEN, "spmv_cases.npz")) as z:
        data = {k: z[k] for k in z.files}
    cases = {}
    for key, arr in data.items():
        name, prec, field = key.rsplit("/", 2)
        cases.setdefault((name, prec), {})[field] = arr
    return cases


@pytest.fixture(scope="session")
def reference():
    """The real reference package — only in the build container."""
    if not os.path.isdir(REFERENCE_SRC):
        pytest.skip("reference sources not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    import mpgmres
    return mpgmres


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def random_sparse(n, density=0.02, shift=4.0, seed=0):
    """Random nonsymmetric dense matrix with a diagonal shift (reference
    tests/conftest.py:20-25 pattern)."""
    r = np.random.default_rng(seed)
    d = r.standard_normal((n, n)) * (r.random((n, n)) < density)
    d += shift * np.eye(n)
    return d


def tridiag(n, lo=-1.0, di=2.0, up=-1.0):
    t = np.zeros((n, n))
    np.fill_diagonal(t, di)
    for i in range(n - 1):
        t[i + 1, i] = lo
        t[i, i + 1] = up
    return t
