import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and the built extension")
    config.addinivalue_line("markers", "slow: longer CPU oracle runs")


@pytest.fixture
def rng():
    # same Philox key as the reference's test fixture (tests/conftest.py:13-15)
    return np.random.Generator(np.random.Philox(key=np.uint64(20240)))


@pytest.fixture(scope="session")
def golden_kernels():
    return np.load(os.path.join(GOLDEN, "kernels.npz"))


@pytest.fixture(scope="session")
def golden_unwrap():
    return np.load(os.path.join(GOLDEN, "unwrap_small.npz"))


@pytest.fixture(scope="session")
def golden_meta():
    import json
    with open(os.path.join(GOLDEN, "golden_meta.json")) as fh:
        return json.load(fh)
