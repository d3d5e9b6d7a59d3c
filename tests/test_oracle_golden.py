"""Pin the CPU oracle (oracle/ibmi_oracle.py) to the reference's own outputs
frozen in tests/golden/ by tests/golden/make_golden.py (which imports the
reference package and asserted bit-equality there)."""

import numpy as np
import pytest

from conftest import golden
from oracle import ibmi_oracle as orc
from paper_2502_06377_b200 import configs, contiguous_partition


def test_oracle_small_solves_bitwise():
    pins = golden("pins.npz")
    for n in range(5):
        a = pins[f"case{n}_a"]
        p, k, f = pins[f"case{n}_pkf"]
        part = contiguous_partition(int(p), int(k), float(f))
        o = orc.solve(a, part.sets, tol=1e-12, max_iterations=60)
        assert np.array_equal(o["result"], pins[f"case{n}_sigma"])
        assert np.array_equal(np.array(o["error_trace"]), pins[f"case{n}_errs"])
        idx, comp = part.sets[0], orc.complement(int(p), part.sets[0])
        s = np.eye(int(p)) + 0.01 * np.ones((int(p), int(p)))
        orc.BlockOp(a, idx, comp).apply(s)
        assert np.array_equal(s, pins[f"case{n}_bu"])
        assert orc.error_estimate(a, s, idx, comp)[0] == pins[f"case{n}_ee"][0]


def test_oracle_not_spd_and_restart():
    pins = golden("pins.npz")
    from paper_2502_06377_b200 import NotPositiveDefinite

    with pytest.raises(NotPositiveDefinite) as ei:
        orc.spd_inverse(pins["notspd_a"])
    assert ei.value.index == pins["notspd_index"][0]
    s, c, it = orc.power_sigma_max(pins["restart_b"])
    assert (s, float(c), float(it)) == tuple(pins["restart_out"])


def test_oracle_c1_full_solve_bitwise():
    g = golden("c1.npz")
    cfg = configs.get_config("c1")
    a = configs.make_matrix("c1")
    o = orc.solve(a, cfg.partition().sets, tol=cfg.tol, max_iterations=cfg.max_iterations, guess="jacobi")
    assert o["iterations"] == int(g["iterations"][0]) == 107
    assert np.array_equal(o["result"], g["sigma"])
    assert np.array_equal(np.array(o["error_trace"]), g["error_trace"])


def test_oracle_c2_first_sweeps():
    g = golden("c2.npz")
    cfg = configs.get_config("c2")
    a = configs.make_matrix("c2")
    o = orc.solve(a, cfg.partition().sets, tol=cfg.tol, max_iterations=2, guess="jacobi", stopping="frobenius")
    assert np.array_equal(np.array(o["error_trace"]), g["error_trace"][:2])
    np.testing.assert_allclose(o["frobenius_trace"], g["frobenius_trace"][:2], rtol=1e-12)


def test_oracle_initial_guesses_against_reference():
    pins = golden("pins.npz")
    a = pins["case1_a"]
    part = contiguous_partition(96, 3, 0.1)
    comp = orc.complement(96, part.sets[0])
    assert np.array_equal(orc.guess_monte_carlo(a, comp, 50, 7), pins["guess_mc"])
    g = pins["guess_takahashi"]
    assert np.abs(orc.guess_takahashi(a, comp) - g).max() <= 1e-12 * np.abs(g).max()


def test_flop_cost_matches_reference():
    from paper_2502_06377_b200.analysis import flop_cost

    pins = golden("pins.npz")
    fc = flop_cost(1000, 4, 0.1)
    assert [fc.m, fc.h, float(fc.total_flops), float(fc.direct_flops)] == pins["an_flop"].tolist()


def test_oracle_nonsymmetric_sigma_against_reference():
    """block_update / error_estimate accept any float64 Σ (solver.py:132-155)."""
    pins = golden("pins.npz")
    a = pins["case2_a"]
    part = contiguous_partition(128, 4, 0.125)
    idx, comp = part.sets[1], orc.complement(128, part.sets[1])
    s = pins["nonsym_sigma0"].copy()
    assert not np.array_equal(s, s.T)
    assert orc.error_estimate(a, s, idx, comp)[0] == pins["nonsym_ee"][0]
    orc.BlockOp(a, idx, comp).apply(s)
    assert np.array_equal(s, pins["nonsym_bu"])


def test_long_fixtures_are_consistent_with_the_pinned_ones():
    """The long reference runs (c4 through its floor, the c2/c3 sketches, c5's first
    sweep on the GPU box's host) repeat the traces of the fixtures the oracle is pinned to."""
    c4, c4l = golden("c4.npz"), golden("c4long.npz")
    assert np.array_equal(c4l["error_trace"][:3], c4["error_trace"][:3])
    assert len(c4l["error_trace"]) == 30 and int(c4l["iterations"][1]) == 0      # the reference never reaches 1e-8
    floor = c4l["error_trace"][25:]
    assert np.all((floor > 3.2e-8) & (floor < 3.4e-8))                            # its FP64 floor
    for it in (3,):
        assert np.array_equal(c4l[f"snap{it}_sample"], c4[f"snap{it}_sample"])
    for name in ("c2", "c3"):
        base, sk = golden(f"{name}.npz"), golden(f"{name}_sketch.npz")
        assert np.array_equal(sk["error_trace"], base["error_trace"])
        assert sk["final_sketch"].shape == (configs.get_config(name).p, 16)
    c5 = golden("c5.npz")
    assert c5["sweep1_sketch"].shape == (65536, 4) and int(c5["power_iters"][0]) == 1598
