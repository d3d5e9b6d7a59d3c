import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (runs through libibmi_b200.so)")
    config.addinivalue_line("markers", "slow: long-running")


def random_spd(p: int, seed: int) -> np.ndarray:
    """Well-conditioned SPD test matrix MᵀM + p·I (reference conftest.py:5-8 recipe)."""
    m = np.random.default_rng(seed).standard_normal((p, p))
    return m.T @ m + p * np.eye(p)


def golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path)


@pytest.fixture
def rng():
    return np.random.default_rng(20248)
