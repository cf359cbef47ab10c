import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the sm_100a library")


def golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


@pytest.fixture(scope="session")
def g_rng():
    return golden("rng.npz")


@pytest.fixture(scope="session")
def g_forward():
    return golden("forward.npz")


@pytest.fixture(scope="session")
def g_chains():
    return golden("chains.npz")


@pytest.fixture(scope="session")
def g_table():
    return golden("table_chains.npz")


@pytest.fixture(scope="session")
def g_energy():
    return golden("energy.npz")


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device (the B200 path has no CPU fallback)")
    torch.cuda.set_device(0)
    return torch.device("cuda", 0)
