import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built extension")


@pytest.fixture
def rng():
    return np.random.default_rng(0)


@pytest.fixture(scope="session")
def golden_lpc():
    return np.load(os.path.join(GOLDEN, "golden_lpc.npz"))


@pytest.fixture(scope="session")
def golden_framewise():
    return np.load(os.path.join(GOLDEN, "golden_framewise.npz"))


@pytest.fixture(scope="session")
def golden_d1():
    return np.load(os.path.join(GOLDEN, "golden_d1.npz"))
