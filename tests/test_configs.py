"""BASELINE problem generators and the algorithmic FLOP model."""

import numpy as np
import pytest

from paper_2502_06377_b200 import configs


def test_flop_model_matches_baseline_table():
    # c1 0.2013 GF, c2 0.1031 TF, c3 1.268 TF, c4 10.147 TF, c5 678.0 TF
    want = {"c1": 0.2013e9, "c2": 0.1031e12, "c3": 1.268e12, "c4": 10.147e12, "c5": 678.0e12}
    for name, v in want.items():
        got = configs.sweep_flops(configs.get_config(name))
        assert abs(got - v) / v < 2e-3, (name, got)
    assert abs(configs.setup_flops(configs.get_config("c4")) - 1.678e12) / 1.678e12 < 2e-3


def test_c1_generator_deterministic_and_spd():
    a = configs.make_matrix("c1", 0)
    b = configs.make_matrix("c1", 0)
    assert np.array_equal(a, b) and np.array_equal(a, a.T)
    w = np.linalg.eigvalsh(a)
    assert 0.99 < w.min() and w.max() < 101


def test_kernel_generator_matches_golden_checksum():
    from conftest import golden

    g = golden("c3.npz")
    a = configs.make_matrix("c3", 0)
    assert np.array_equal(a, a.T)
    np.testing.assert_allclose(g["a_checksum"], [a.sum(), np.linalg.norm(a), a[0, 0], a[-1, -1]], rtol=1e-13)


def test_c5_not_on_host():
    with pytest.raises(ValueError):
        configs.make_matrix("c5")
