import os
import sys

import numpy as np
import pytest
from threadpoolctl import threadpool_limits

# single-threaded BLAS/LAPACK for the oracle: multi-threaded eigh/solve reductions
# change rounding with machine load, which can flip near-zero PSD clamps
_BLAS_LIMIT = threadpool_limits(limits=1)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, GOLDEN):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def load(name):
        if name not in cache:
            cache[name] = dict(np.load(os.path.join(GOLDEN, name)))
        return cache[name]

    return load


def rel_err(a, b, tiny=1e-300):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), tiny))
