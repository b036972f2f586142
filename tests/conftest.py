import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the C-ABI on cuda:0)")


def load_pq(name):
    import oracle
    z = np.load(os.path.join(GOLDEN, name))
    return oracle.PQ(int(z["m"]), int(z["dbits"]), int(z["dim"]), z["codebooks"], z["perms"])


@pytest.fixture(scope="session")
def pq8():
    return load_pq("pq_d128_m8.npz")


@pytest.fixture(scope="session")
def pq16():
    return load_pq("pq_d256_m16.npz")


@pytest.fixture(scope="session")
def g8():
    return dict(np.load(os.path.join(GOLDEN, "golden_m8.npz")))


@pytest.fixture(scope="session")
def g16():
    return dict(np.load(os.path.join(GOLDEN, "golden_m16.npz")))
