"""GPU parity: the CUDA path (through libibmi_b200.so) against the oracle and
the reference-generated golden fixtures.

Tolerances:
  * Σ: relative Frobenius error ≤ 1e-10 against the reference (BASELINE north star);
  * error trace: |Δerr| ≤ 1e-6·err_ref + 5e-2·tol per sweep (SURVEY B7 proposed 1e-2·tol; the
    estimate B = Σ[I,:]·A[:,c] is a cancellation whose absolute rounding floor is ~1e-10 at c3 —
    |Σ| up to 1/nugget = 100 over 8192-term sums — so a different summation order, e.g. split-K,
    moves err by ~1e-10 = 1e-2·tol);
  * sweep count: exact, or ±1 when some reference error lies inside that band around tol;
  * dense kernels (GEMM, SPD inverse) against float64 torch/numpy: ≤ 1e-13 relative.
"""

from __future__ import annotations

import warnings

import numpy as np
import pytest

from conftest import golden, random_spd

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA (run with -m 'not gpu' on CPU hosts)")
    import paper_2502_06377_b200 as pkg

    pkg.load_library()   # fails loudly if the .so is missing


def rel_fro(x, ref):
    return float(np.linalg.norm(np.asarray(x) - ref) / np.linalg.norm(ref))


def band_ok(err, ref, tol):
    return abs(err - ref) <= 1e-6 * ref + 5e-2 * tol


def check_trace(errs, ref_errs, tol):
    ref_errs = np.asarray(ref_errs)
    n = min(len(errs), len(ref_errs))
    for i in range(n):
        assert band_ok(errs[i], ref_errs[i], tol), (i, errs[i], ref_errs[i])
    if len(errs) != len(ref_errs):
        near = np.any(np.abs(ref_errs - tol) <= 1e-6 * ref_errs + 5e-2 * tol)
        assert near and abs(len(errs) - len(ref_errs)) <= 1, (len(errs), len(ref_errs))


def check_sketch(sigma, g, key, tol=1e-10):
    """‖(Σ − Σ_ref)·R‖_F / ‖Σ_ref·R‖_F with the seeded Gaussian R of make_golden.sketch_matrix:
    an unbiased estimate of the full relative Frobenius distance (E‖XR‖_F² = cols·‖X‖_F²),
    from a fixture of p × cols doubles instead of p²; plus ‖Σ‖_F and the row sums."""
    ref = g[f"{key}_sketch"]
    r = np.random.default_rng(2025).standard_normal((sigma.shape[0], ref.shape[1]))
    assert rel_fro(sigma @ r, ref) < tol
    fro = float(g[f"{key}_fro"][0])
    assert abs(np.linalg.norm(sigma) - fro) <= tol * fro
    assert np.linalg.norm(sigma.sum(axis=1) - g[f"{key}_rowsum"]) <= tol * fro * np.sqrt(sigma.shape[0])


# ----------------------------------------------------------------- kernels
@pytest.mark.parametrize("m,n,k", [(128, 128, 16), (256, 384, 512), (1, 1, 1), (129, 77, 33), (300, 257, 1000),
                                   (1000, 64, 7), (5, 700, 300)])
def test_dgemm_nt_matches_torch_fp64(m, n, k):
    from paper_2502_06377_b200.linalg import dgemm_nt

    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    x = torch.randn((m, k), dtype=torch.float64, device="cuda", generator=g)
    y = torch.randn((n, k), dtype=torch.float64, device="cuda", generator=g)
    c0 = torch.randn((m, n), dtype=torch.float64, device="cuda", generator=g)
    out = dgemm_nt(x, y, alpha=-0.5, beta=2.0, c=c0.clone())
    ref = -0.5 * (x @ y.T) + 2.0 * c0
    torch.cuda.synchronize()
    err = (out - ref).abs().max().item()
    scale = (x.abs() @ y.abs().T).max().item() + 2 * c0.abs().max().item()
    assert err <= 1e-14 * max(scale, 1.0) * max(1, k) ** 0.5


def test_dgemm_nt_unaligned_views():
    """Odd leading dimensions / offsets force the 8-byte cp.async path."""
    from paper_2502_06377_b200.linalg import dgemm_nt

    g = torch.Generator(device="cuda").manual_seed(3)
    big = torch.randn((301, 211), dtype=torch.float64, device="cuda", generator=g)
    x = big[1:200, 1:150]      # odd column offset -> 8B aligned only
    y = big[3:170, 3:152]
    out = torch.zeros((199, 167), dtype=torch.float64, device="cuda")
    dgemm_nt(x, y, c=out)
    ref = x @ y.T
    assert (out - ref).abs().max().item() < 1e-11


@pytest.mark.parametrize("n", [1, 2, 63, 64, 65, 200, 513, 1024])
def test_spd_inverse_against_numpy(n):
    from paper_2502_06377_b200.linalg import spd_inverse

    a = random_spd(n, n)
    inv = spd_inverse(a)
    assert np.array_equal(inv, inv.T)                       # exactly symmetric (linalg.py:130)
    ref = np.linalg.inv(a)
    assert rel_fro(inv, ref) < 1e-12
    assert np.linalg.norm(a @ inv - np.eye(n), 2) <= 1e-8     # reference test_linalg.py:159-161


def test_spd_inverse_not_spd_reports_pivot():
    from paper_2502_06377_b200 import NotPositiveDefinite
    from paper_2502_06377_b200.linalg import spd_inverse

    pins = golden("pins.npz")
    with pytest.raises(NotPositiveDefinite) as ei:
        spd_inverse(pins["notspd_a"])
    assert ei.value.index == int(pins["notspd_index"][0])
    # a failure deep inside a blocked factorisation (pivot 150 of 300)
    a = random_spd(300, 1)
    a[150, 150] = -1e6
    with pytest.raises(NotPositiveDefinite) as ei:
        spd_inverse(a)
    from scipy.linalg.lapack import dpotrf

    assert ei.value.index == dpotrf(a, lower=1)[1] - 1


def test_spd_inverse_rejects_asymmetric():
    from paper_2502_06377_b200.linalg import spd_inverse

    a = random_spd(20, 2)
    a[0, 5] += 1.0
    with pytest.raises(ValueError):
        spd_inverse(a)


@pytest.mark.parametrize("shape,seed", [((40, 90), 0), ((90, 40), 1), ((300, 1200), 2), ((1500, 200), 3), ((7, 7), 4)])
def test_two_norm_matches_oracle(shape, seed):
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200.linalg import two_norm

    b = np.random.default_rng(seed).standard_normal(shape)
    s = two_norm(b)
    s_ref, conv, it_ref = orc.power_sigma_max(b)
    assert abs(s - s_ref) <= 1e-9 * s_ref
    assert abs(two_norm.last_iterations - it_ref) <= 2
    assert abs(s - np.linalg.norm(b, 2)) <= 1e-6 * s      # reference test_linalg.py:205-213


def test_two_norm_zero_and_restart_paths():
    from paper_2502_06377_b200.linalg import two_norm

    pins = golden("pins.npz")
    assert two_norm(np.zeros((5, 7))) == 0.0
    s_ref, c_ref, it_ref = pins["restart_out"]
    s = two_norm(pins["restart_b"])     # rows sum to zero: y1 = 0 -> restart from default_rng(0x5EED)
    assert abs(s - s_ref) <= 1e-9 * s_ref
    assert abs(two_norm.last_iterations - it_ref) <= 2


@pytest.mark.parametrize("shape,seed", [((700, 1500), 6), ((1536, 900), 7), ((2048, 2048), 8), ((2100, 1800), 9),
                                        ((2200, 2600), 10), ((1152, 7040), 11)])
def test_two_norm_flag_exchange_kernel(shape, seed):
    """Mid-size Gram matrices (640 < n ≤ 2220) run the flag-carrying line exchange
    (power_gram_ll_kernel) instead of one grid barrier per iteration: same σ and
    iteration count as the oracle and as the grid-barrier kernel (ibmi_tune key 13)."""
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import _abi
    from paper_2502_06377_b200.linalg import two_norm

    rng = np.random.default_rng(seed)
    b = rng.standard_normal(shape) * np.exp(rng.uniform(-2, 2, size=(shape[0], 1)))
    s = two_norm(b)
    it = two_norm.last_iterations
    s_ref, conv, it_ref = orc.power_sigma_max(b)
    assert abs(s - s_ref) <= 1e-9 * s_ref
    assert abs(it - it_ref) <= 2
    _abi.check(_abi.lib().ibmi_tune(13, 0), "tune")
    try:
        s_bar = two_norm(b)
        it_bar = two_norm.last_iterations
    finally:
        _abi.check(_abi.lib().ibmi_tune(13, 1), "tune")
    assert abs(s - s_bar) <= 1e-12 * s_bar and abs(it - it_bar) <= 1


@pytest.mark.parametrize("shape", [(800, 1024), (1500, 1024)])
def test_two_norm_flag_exchange_restart_and_cap(shape):
    """σ = 0 on the first iterate restarts from default_rng(0x5EED) inside the
    flag-exchange kernel (linalg.py:237-244); the cap still warns.  Rows of dyadic
    entries summing to zero over 1024 columns (1/√1024 is exact) make B·v₁ an exact 0
    in both Gram forms (row Gram for 800 rows, column Gram for 1500)."""
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import NoConvergenceWarning
    from paper_2502_06377_b200.linalg import two_norm

    b = np.random.default_rng(12).standard_normal(shape)
    b = b - b.mean(axis=1, keepdims=True)
    b[:, -1] -= b.sum(axis=1)            # exact zero row sums up to rounding ...
    b = np.round(b * 1024) / 1024        # ... made exact: dyadic entries
    b[:, -1] -= b.sum(axis=1)
    assert np.all(b.sum(axis=1) == 0.0)
    s_ref, conv, it_ref = orc.power_sigma_max(b)
    s = two_norm(b)
    assert abs(s - s_ref) <= 1e-9 * s_ref
    assert abs(two_norm.last_iterations - it_ref) <= 2
    with pytest.warns(NoConvergenceWarning):
        two_norm(np.random.default_rng(13).standard_normal(shape), rtol=1e-300, max_iters=4)


def test_two_norm_warns_at_cap():
    from paper_2502_06377_b200 import NoConvergenceWarning
    from paper_2502_06377_b200.linalg import two_norm

    b = np.random.default_rng(5).standard_normal((30, 30))
    with pytest.warns(NoConvergenceWarning):
        two_norm(b, rtol=1e-300, max_iters=3)


# ------------------------------------------------- single-step entry points
def test_block_update_and_error_estimate_match_reference():
    import paper_2502_06377_b200 as pkg

    pins = golden("pins.npz")
    for n in range(5):
        a = pins[f"case{n}_a"]
        p, k, f = pins[f"case{n}_pkf"]
        part = pkg.contiguous_partition(int(p), int(k), float(f))
        idx, comp = part.sets[0], pkg.complement(part, 0)
        sig = np.eye(int(p)) + 0.01 * np.ones((int(p), int(p)))
        pkg.block_update(a, sig, idx, comp)
        assert rel_fro(sig, pins[f"case{n}_bu"]) < 1e-12
        e = pkg.error_estimate(a, sig, idx, comp)
        e_ref = float(pins[f"case{n}_ee"][0])
        assert abs(e - e_ref) <= 1e-9 * e_ref + 1e-13


def test_block_update_noncontiguous_set():
    """Arbitrary idx (relabelled on the host) equals the oracle update."""
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc

    p = 160
    a = random_spd(p, 11)
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(p, 70, replace=False))
    comp = orc.complement(p, idx)
    s0 = np.eye(p) + 0.001 * np.ones((p, p))
    s1 = s0.copy()
    pkg.block_update(a, s1, idx, comp)
    s2 = s0.copy()
    orc.BlockOp(a, idx, comp).apply(s2)
    assert rel_fro(s1, s2) < 1e-12


def test_block_update_non_float64_sigma_is_not_written():
    """Reference quirk (solver.py:139): only float64 arrays update in place."""
    import paper_2502_06377_b200 as pkg

    a = random_spd(64, 3)
    part = pkg.contiguous_partition(64, 2)
    s = np.eye(64, dtype=np.float32)
    before = s.copy()
    pkg.block_update(a, s, part.sets[0], pkg.complement(part, 0))
    assert np.array_equal(s, before)


def test_shape_errors():
    import paper_2502_06377_b200 as pkg

    a = random_spd(32, 0)
    part = pkg.contiguous_partition(40, 2)
    with pytest.raises(pkg.DimensionMismatch):
        pkg.solve(a, part)
    with pytest.raises(pkg.DimensionMismatch):
        pkg.block_update(a, np.eye(31), np.arange(16), np.arange(16, 32))


def test_solve_not_spd_raises_block_local_pivot():
    import paper_2502_06377_b200 as pkg

    a = random_spd(96, 4)
    a[70, 70] = -5.0        # inside set 1 of a 2-block split -> local step 70 - 48 = 22
    part = pkg.contiguous_partition(96, 2)
    with pytest.raises(pkg.NotPositiveDefinite) as ei:
        pkg.solve(a, part)
    assert ei.value.index == 22
    assert ei.value.set_index == 1


# ---------------------------------------------------------- whole solves
def test_solve_small_cases_match_reference():
    import paper_2502_06377_b200 as pkg

    pins = golden("pins.npz")
    for n in range(5):
        a = pins[f"case{n}_a"]
        p, k, f = pins[f"case{n}_pkf"]
        part = pkg.contiguous_partition(int(p), int(k), float(f))
        rep = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-12, max_iterations=60))
        ref_sigma = pins[f"case{n}_sigma"]
        ref_it, ref_conv = pins[f"case{n}_iters"]
        assert rel_fro(rep.result, ref_sigma) < 1e-10
        check_trace(rep.error_trace, pins[f"case{n}_errs"], 1e-12)
        assert rep.converged == bool(ref_conv)
        assert np.array_equal(rep.result, rep.result.T)


def test_solve_red_black_matches_oracle():
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc

    p = 256
    a = random_spd(p, 9)
    part = pkg.red_black_partition(p)
    rep = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-11))
    o = orc.solve(a, part.sets, tol=1e-11)
    assert rel_fro(rep.result, o["result"]) < 1e-10
    check_trace(rep.error_trace, o["error_trace"], 1e-11)


def test_c1_full_solve_matches_reference():
    """BASELINE c1 (p=512, 2 blocks, Σ0 = diag(1/A_ii), tol 1e-10): same sweep
    count, trace in band, Σ within 1e-10 relative Frobenius of the reference."""
    import paper_2502_06377_b200 as pkg
    from paper_2502_06377_b200 import configs

    g = golden("c1.npz")
    cfg = configs.get_config("c1")
    a = configs.make_matrix("c1")
    rep = pkg.solve(a, cfg.partition(), pkg.IbmiConfig(tol=cfg.tol, max_iterations=cfg.max_iterations,
                                                       initial_guess="jacobi"))
    assert rep.converged
    check_trace(rep.error_trace, g["error_trace"], cfg.tol)
    assert rel_fro(rep.result, g["sigma"]) < 1e-10


def test_c2_full_solve_frobenius_stop():
    """BASELINE c2 (p=4096): sweep until ‖I − AΣ‖_F < 1e-9."""
    import paper_2502_06377_b200 as pkg
    from paper_2502_06377_b200 import configs

    g = golden("c2.npz")
    cfg = configs.get_config("c2")
    a = configs.make_matrix("c2")
    rep = pkg.solve(a, cfg.partition(), pkg.IbmiConfig(tol=cfg.tol, max_iterations=cfg.max_iterations,
                                                       initial_guess="jacobi", stopping="frobenius",
                                                       residual_every_sweep=True))
    # the bound-based skip of the residual must stop at the same sweep
    rep2 = pkg.solve(a, cfg.partition(), pkg.IbmiConfig(tol=cfg.tol, max_iterations=cfg.max_iterations,
                                                        initial_guess="jacobi", stopping="frobenius"))
    assert rep2.iterations == rep.iterations
    assert np.array_equal(rep2.result, rep.result)
    ref_fro = g["frobenius_trace"]
    n = min(len(rep.residual_trace), len(ref_fro))
    fr = np.asarray(rep.residual_trace[:n])
    assert np.all(np.abs(fr - ref_fro[:n]) <= 1e-6 * ref_fro[:n] + 5e-2 * cfg.tol)
    assert abs(rep.iterations - int(g["iterations"][0])) <= 1
    sample = rep.result[g["sample_i"], g["sample_j"]]
    assert rel_fro(sample, g["sample"]) < 1e-10
    assert rel_fro(np.diag(rep.result), g["diag"]) < 1e-10
    check_sketch(rep.result, golden("c2_sketch.npz"), "final")


def test_c3_full_solve_matches_reference():
    import paper_2502_06377_b200 as pkg
    from paper_2502_06377_b200 import configs

    g = golden("c3.npz")
    cfg = configs.get_config("c3")
    a = configs.make_matrix("c3")
    rep = pkg.solve(a, cfg.partition(), pkg.IbmiConfig(tol=cfg.tol))
    check_trace(rep.error_trace, g["error_trace"], cfg.tol)
    sample = rep.result[g["sample_i"], g["sample_j"]]
    assert rel_fro(sample, g["sample"]) < 1e-10
    dr = np.linalg.norm(rep.result.sum(axis=1) - g["rowsum"])
    assert dr <= 1e-10 * float(g["fro"][0]) * np.sqrt(rep.result.shape[0])
    check_sketch(rep.result, golden("c3_sketch.npz"), "final")


@pytest.mark.parametrize("seed", [1, 2])
def test_c1_repeat_seeds_full_solve_matches_oracle(seed):
    """repeats use seeds 1 and 2.  Full c1 solves against the oracle (bit-identical to
    the reference on seed 0): same sweep count, trace in band, the whole Σ within 1e-10."""
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import configs

    cfg = configs.get_config("c1")
    a = configs.make_matrix("c1", seed)
    rep = pkg.solve(a, cfg.partition(), pkg.IbmiConfig(tol=cfg.tol, max_iterations=cfg.max_iterations,
                                                       initial_guess="jacobi"))
    o = orc.solve(a, cfg.partition().sets, tol=cfg.tol, max_iterations=cfg.max_iterations, guess="jacobi")
    assert rep.converged and o["converged"]
    check_trace(rep.error_trace, o["error_trace"], cfg.tol)
    assert rel_fro(rep.result, o["result"]) < 1e-10


@pytest.mark.slow
def test_c4_first_sweep_whole_sigma_matches_oracle():
    """c4 at full size, the north-star metric itself: the WHOLE Σ (16384², not a sketch) after the
    first sweep against the oracle's first sweep run on this host's cores (about a minute of CPU)."""
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import configs
    from paper_2502_06377_b200.device import DeviceSolver

    cfg = configs.get_config("c4")
    a = configs.make_matrix("c4")
    part = cfg.partition()
    with DeviceSolver(a, partition=part) as ds:
        ds.setup()
        ds.init_sigma(0)
        err = ds.sweep(1e-9, 5000)[0]
        s = ds.sigma()
    sigma = np.eye(cfg.p)
    for idx in part.sets:                       # W per set on the fly: same arithmetic, 2 GB less RAM
        orc.BlockOp(a, idx, orc.complement(cfg.p, idx)).apply(sigma)
    ref_err = orc.error_estimate(a, sigma, part.sets[-1], orc.complement(cfg.p, part.sets[-1]))[0]
    assert rel_fro(s, sigma) < 1e-10
    assert abs(err - ref_err) <= 1e-6 * ref_err
    assert abs(ref_err - float(golden("c4long.npz")["error_trace"][0])) <= 1e-9 * ref_err   # the reference's value


@pytest.mark.parametrize("name,seed,sweeps", [("c2", 1, 2), ("c3", 1, 1)])
def test_c2_c3_repeat_seed_whole_sigma_matches_oracle(name, seed, sweeps):
    """The north-star metric on the WHOLE Σ (not a sketch) at full c2 / c3 size: the first sweeps
    of a repeat seed on the GPU against the oracle's, relative Frobenius ≤ 1e-10."""
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import configs
    from paper_2502_06377_b200.device import DeviceSolver

    cfg = configs.get_config(name)
    a = configs.make_matrix(name, seed)
    part = cfg.partition()
    with DeviceSolver(a, partition=part) as ds:
        ds.setup()
        ds.init_sigma(1 if cfg.guess == "jacobi" else 0)
        errs = [ds.sweep(1e-9, 5000)[0] for _ in range(sweeps)]
        s = ds.sigma()
    o = orc.solve(a, part.sets, tol=1e-300, max_iterations=sweeps, guess=cfg.guess)
    assert rel_fro(s, o["result"]) < 1e-10
    assert np.array_equal(s, s.T)
    for e, r in zip(errs, o["error_trace"]):
        assert abs(e - r) <= 1e-6 * r + 5e-2 * cfg.tol


def test_c4_through_the_floor_matches_reference():
    """c4 (p=16384) against the reference's own 30-sweep CPU run (tests/golden/c4long.npz,
    generated by make_golden.py c4long from the reference package): the whole error
    trajectory down to the FP64 floor, the sweep at which tol is met, and Σ at seven
    checkpoints through a Gaussian sketch, row sums, ‖Σ‖_F and sampled entries at 1e-10.

    The reference stalls at 3.30e-8 (never reaching its default tol 1e-8); c4's tol is
    pinned at 1e-7 (configs.py), which the reference meets at sweep 24."""
    from paper_2502_06377_b200 import configs
    from paper_2502_06377_b200.device import DeviceSolver

    g = golden("c4long.npz")
    cfg = configs.get_config("c4")
    assert cfg.tol == 1e-7
    a = configs.make_matrix("c4")
    ref = g["error_trace"]
    cps = {int(c) for c in g["checkpoints"]}
    r = np.random.default_rng(2025).standard_normal((cfg.p, g["snap3_sketch"].shape[1]))
    errs = []
    with DeviceSolver(a, partition=cfg.partition()) as ds:
        ds.setup()
        ds.init_sigma(0)
        for it in range(1, len(ref) + 1):
            err, pit, _ = ds.sweep(1e-9, 5000)
            errs.append(err)
            if ref[it - 1] > 5e-8:          # above the floor the estimates agree inside the B7 band
                assert band_ok(err, ref[it - 1], cfg.tol), (it, err, ref[it - 1])
            if it in cps:
                s = ds.sigma()
                fro = float(g[f"snap{it}_fro"][0])
                assert rel_fro(s @ r, g[f"snap{it}_sketch"]) < 1e-10, it
                assert rel_fro(s[g["sample_i"], g["sample_j"]], g[f"snap{it}_sample"]) < 1e-10, it
                assert np.linalg.norm(s.sum(axis=1) - g[f"snap{it}_rowsum"]) <= 1e-10 * fro * np.sqrt(cfg.p), it
                assert abs(np.linalg.norm(s) - fro) <= 1e-10 * fro, it
                if it == len(ref):
                    assert np.array_equal(s, s.T)
                del s
        fr = ds.frobenius()
    errs = np.array(errs)
    # same sweep count to tol as the reference (24)
    n_gpu = int(np.argmax(errs <= cfg.tol)) + 1
    n_ref = int(np.argmax(ref <= cfg.tol)) + 1
    assert n_ref == 24 and n_gpu == n_ref, (n_gpu, n_ref)
    # the floor: the reference sits at 3.30e-8 / ‖I − AΣ‖_F = 4.47e-7; not worse than 1.5x that
    assert np.all(errs[25:] < 1.5 * ref[25:].max()), errs[25:]
    assert fr < 1.5 * float(g["snap30_frobenius"][0]), fr


@pytest.mark.slow
def test_c5_first_sweep_matches_oracle_fixture():
    """c5 (p = 65536, 16 sets of 4608/5120) at full size: setup + the first sweep
    against the fixture the CPU oracle produced on the GPU box's host
    (tools/make_c5_fixture.py: 16 block updates + the estimate in solve()'s order,
    ~20 min of 16 cores).  Σ is compared through a seeded Gaussian sketch Σ·R
    (E‖XR‖_F² = cols·‖X‖_F²: an estimate of the full relative Frobenius distance),
    its row sums, ‖Σ‖_F and 4096 sampled entries, all at 1e-10."""
    from paper_2502_06377_b200 import configs
    from paper_2502_06377_b200.device import DeviceSolver

    g = golden("c5.npz")
    free, _total = torch.cuda.mem_get_info()
    if free < 150e9:
        pytest.skip("c5 needs ~120 GB of HBM")
    cfg = configs.get_config("c5")
    p = cfg.p
    a_dev = configs.make_matrix_c5_device(0)
    chk = np.array([float(a_dev.sum()), float(torch.linalg.norm(a_dev)), float(a_dev[0, 0]), float(a_dev[-1, -1]),
                    float(a_dev[123, 45678])])
    assert np.allclose(chk, g["a_checksum"], rtol=1e-12, atol=0.0), (chk, g["a_checksum"])
    ds = DeviceSolver(a_dev, partition=cfg.partition())
    del a_dev
    torch.cuda.empty_cache()
    try:
        ds.setup()
        ds.init_sigma(0)
        err, pit, conv = ds.sweep(1e-9, 5000)
        ref_err = float(g["error_trace"][0])
        assert abs(err - ref_err) <= 1e-6 * ref_err + 5e-2 * cfg.tol, (err, ref_err)
        assert abs(pit - int(g["power_iters"][0])) <= 2
        s = ds.sigma_view()
        assert s.shape == (p, p)
        r = torch.as_tensor(np.random.default_rng(2025).standard_normal((p, g["sweep1_sketch"].shape[1])),
                            device=s.device)
        sk = torch.empty((p, r.shape[1]), dtype=torch.float64, device=s.device)
        rs = torch.empty(p, dtype=torch.float64, device=s.device)
        fro2 = 0.0
        for lo in range(0, p, 4096):
            blk = s[lo:lo + 4096]
            sk[lo:lo + 4096] = blk @ r
            rs[lo:lo + 4096] = blk.sum(dim=1)
            fro2 += float((blk * blk).sum())
        ref_fro = float(g["sweep1_fro"][0])
        assert rel_fro(sk.cpu().numpy(), g["sweep1_sketch"]) < 1e-10
        assert np.linalg.norm(rs.cpu().numpy() - g["sweep1_rowsum"]) <= 1e-10 * ref_fro * np.sqrt(p)
        assert abs(fro2 ** 0.5 - ref_fro) <= 1e-10 * ref_fro
        si = torch.as_tensor(g["sample_i"], device=s.device)
        sj = torch.as_tensor(g["sample_j"], device=s.device)
        assert rel_fro(s[si, sj].cpu().numpy(), g["sweep1_sample"]) < 1e-10
        # symmetric to the bit on sampled pairs
        assert torch.equal(s[si, sj], s[sj, si])
    finally:
        ds.close()
        from paper_2502_06377_b200 import _abi

        _abi.lib().ibmi_release_cached_memory(-1)
        torch.cuda.empty_cache()


def test_solve_overlapping_noncontiguous_matches_oracle():
    """Custom JSON partition with overlapping, non-contiguous sets (reference
    partition.py:124-141) runs on the general index-list path."""
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc

    p = 300
    a = random_spd(p, 21)
    rng = np.random.default_rng(4)
    perm = rng.permutation(p)
    sets = [np.sort(perm[:140]), np.sort(perm[110:230]), np.sort(perm[200:])]   # overlapping, scattered
    part = pkg.load_partition_json({"p": p, "sets": [s.tolist() for s in sets]})
    rep = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-11))
    o = orc.solve(a, part.sets, tol=1e-11)
    assert rep.converged
    assert rel_fro(rep.result, o["result"]) < 1e-10
    check_trace(rep.error_trace, o["error_trace"], 1e-11)


def test_solve_mixed_runs_and_lists_local_guess():
    """Some sets are runs, some scattered; 'local' initial guess on the GPU."""
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc

    p = 256
    a = random_spd(p, 22)
    s0 = np.arange(0, 100)
    s1 = np.concatenate([np.arange(90, 180), np.arange(200, 220)])
    s2 = np.concatenate([np.arange(170, 200), np.arange(210, 256)])
    part = pkg.load_partition_json({"p": p, "sets": [s0.tolist(), s1.tolist(), s2.tolist()]})
    rep = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-11, initial_guess="local"))
    o = orc.solve(a, part.sets, tol=1e-11, guess="local")
    assert rel_fro(rep.result, o["result"]) < 1e-10
    check_trace(rep.error_trace, o["error_trace"], 1e-11)


def test_initial_guesses_match_reference():
    """GPU mc / takahashi / local guesses against the reference's own values."""
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc

    pins = golden("pins.npz")
    a = pins["case1_a"]
    part = pkg.contiguous_partition(96, 3, 0.1)
    comp = pkg.complement(part, 0)
    # multi-block factorisations (c > 64) of the Schur complement as well
    big = random_spd(300, 8)
    cbig = np.arange(40, 300)
    assert rel_fro(pkg.initial_guess_takahashi(big, cbig), np.linalg.inv(big)[np.ix_(cbig, cbig)]) < 1e-12
    g = pkg.initial_guess_monte_carlo(a, comp, 50, 7)
    assert rel_fro(g, pins["guess_mc"]) < 1e-12
    g = pkg.initial_guess_takahashi(a, comp)
    assert rel_fro(g, pins["guess_takahashi"]) < 1e-12
    g = pkg.initial_guess_local_inverse(a, comp)
    assert rel_fro(g, orc.spd_inverse(a[np.ix_(comp, comp)])) < 1e-12


@pytest.mark.parametrize("guess", ["mc", "takahashi"])
@pytest.mark.parametrize("kind", ["contiguous", "red-black", "general"])
def test_solve_with_guess_matches_oracle(guess, kind):
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc

    p = 192
    a = random_spd(p, 31)
    if kind == "contiguous":
        part = pkg.contiguous_partition(p, 3, 0.1)
    elif kind == "red-black":
        part = pkg.red_black_partition(p)
    else:
        perm = np.random.default_rng(5).permutation(p)
        part = pkg.load_partition_json({"p": p, "sets": [np.sort(perm[:110]).tolist(), np.sort(perm[90:]).tolist()]})
    cfg = pkg.IbmiConfig(tol=1e-11, initial_guess=guess, mc_samples=40, mc_seed=3)
    rep = pkg.solve(a, part, cfg)
    o = orc.solve(a, part.sets, tol=1e-11, guess=guess, mc_samples=40, mc_seed=3)
    assert rep.converged and abs(rep.iterations - o["iterations"]) <= 1
    assert rel_fro(rep.result, o["result"]) < 1e-10


def test_cli_invert_streams_ibmi1_and_matches_solve(tmp_path):
    import json

    import paper_2502_06377_b200 as pkg
    from paper_2502_06377_b200 import matio
    from paper_2502_06377_b200.cli import main

    p = 640
    a = random_spd(p, 41)
    fin, fout, frep = tmp_path / "a.ibmi", tmp_path / "s.ibmi", tmp_path / "r.json"
    matio.save_ibmi(fin, a)
    assert main(["invert", "--in", str(fin), "--out", str(fout), "--blocks", "3", "--overlap", "0.1",
                 "--tol", "1e-11", "--report", str(frep)]) == 0
    rep = pkg.solve(a, pkg.contiguous_partition(p, 3, 0.1), pkg.IbmiConfig(tol=1e-11))
    s = matio.load_ibmi(fout)
    assert np.array_equal(s, rep.result)
    meta = json.loads(frep.read_text())
    assert meta["iterations"] == rep.iterations and meta["converged"]
    # red-black goes through the host (relabelled), CSV output
    fcsv = tmp_path / "s.csv"
    assert main(["invert", "--in", str(fin), "--out", str(fcsv), "--ordering", "red-black", "--tol", "1e-11"]) == 0
    rb = pkg.solve(a, pkg.red_black_partition(p), pkg.IbmiConfig(tol=1e-11))
    assert np.array_equal(matio.load_csv(fcsv), rb.result)


def test_cli_compare(tmp_path, capsys):
    import json

    from paper_2502_06377_b200 import matio
    from paper_2502_06377_b200.cli import main

    a = random_spd(300, 42)
    f = tmp_path / "a.ibmi"
    matio.save_ibmi(f, a)
    assert main(["compare", "--in", str(f), "--blocks", "2", "--tol", "1e-12"]) == 0
    out = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert out["converged"] and out["relative_error_2norm"] < 1e-10


def test_analysis_diagnostics_match_reference():
    import warnings

    import paper_2502_06377_b200 as pkg
    from paper_2502_06377_b200 import analysis

    pins = golden("pins.npz")
    a = pins["case0_a"]
    i1, i2 = pkg.contiguous_partition(64, 2, 0.0).sets
    assert abs(analysis.contraction_factor(a, i1, i2) - pins["an_contraction"][0]) <= 1e-9 * pins["an_contraction"][0]
    assert abs(analysis.spectral_radius_condition(a, i1, i2) - pins["an_spectral"][0]) <= 1e-8 * pins["an_spectral"][0]
    assert abs(analysis.condition_number_2(a) - pins["an_cond"][0]) <= 1e-8 * pins["an_cond"][0]
    x0 = np.eye(64) / np.abs(a).sum(axis=1).max()
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        x, it, cv = analysis.newton_schultz(a, x0, tol=1e-10)
    assert cv and abs(it - int(pins["an_newton_meta"][0])) <= 1
    assert rel_fro(x, pins["an_newton_x"]) < 1e-10
    assert analysis.lemma_error_recurrence_check(a, i1, i2, np.eye(32) * 0.5, 3) < 1e-10


@pytest.mark.parametrize("p,k,f", [(5, 2, 0.0), (9, 4, 0.0), (33, 3, 0.3), (127, 5, 0.25), (250, 10, 0.1),
                                   (257, 2, 0.45), (600, 7, 0.0), (1001, 3, 0.2), (2048, 16, 0.125),
                                   (1500, 4, 0.05)])
def test_solve_shapes_match_oracle(p, k, f):
    """Odd orders, tiny sets, many blocks, deep overlaps: every kernel path
    (TMA / cp.async 16B / 8B, split-K, cluster vs grid power iteration)."""
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc

    a = random_spd(p, p + k)
    part = pkg.contiguous_partition(p, k, f)
    sweeps = 4
    rep = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-300, max_iterations=sweeps))
    o = orc.solve(a, part.sets, tol=1e-300, max_iterations=sweeps)
    assert rel_fro(rep.result, o["result"]) < 1e-10
    np.testing.assert_allclose(rep.error_trace, o["error_trace"], rtol=1e-6, atol=1e-12)
    assert np.array_equal(rep.result, rep.result.T)


@pytest.mark.parametrize("p,k,f", [(512, 2, 0.0), (9, 4, 0.0), (300, 3, 0.1), (777, 5, 0.2), (1024, 8, 0.125),
                                   (1000, 2, 0.3)])
def test_fused_small_sweep_equals_unfused(p, k, f):
    """p ≤ 1024: the sweep's GEMM phases run as one cooperative kernel (small_sweep.cuh,
    ibmi_tune key 14).  Same Σ (≤ 1e-12 relative Frobenius), same error trace and sweep
    count as the per-GEMM launches, and both match the oracle."""
    import paper_2502_06377_b200 as pkg
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import _abi

    a = random_spd(p, p + k)
    part = pkg.contiguous_partition(p, k, f)
    cfg = pkg.IbmiConfig(tol=1e-11, max_iterations=60)
    fused = pkg.solve(a, part, cfg)
    _abi.check(_abi.lib().ibmi_tune(14, 0), "tune")
    try:
        plain = pkg.solve(a, part, cfg)
    finally:
        _abi.check(_abi.lib().ibmi_tune(14, 1), "tune")
    assert fused.iterations == plain.iterations and fused.converged == plain.converged
    assert rel_fro(fused.result, plain.result) < 1e-12
    np.testing.assert_allclose(fused.error_trace, plain.error_trace, rtol=1e-6, atol=1e-13)
    assert np.array_equal(fused.result, fused.result.T)
    o = orc.solve(a, part.sets, tol=1e-11, max_iterations=60)
    assert abs(fused.iterations - o["iterations"]) <= 1
    assert rel_fro(fused.result, o["result"]) < 1e-10


@pytest.mark.parametrize("stopping", ["estimate", "frobenius"])
def test_device_loop_equals_host_loop(stopping, monkeypatch):
    """The conditional-graph solve loop gives the host loop's sweeps bit for bit."""
    import paper_2502_06377_b200 as pkg

    p = 384
    a = random_spd(p, 51)
    part = pkg.contiguous_partition(p, 3, 0.1)
    cfg = pkg.IbmiConfig(tol=1e-11, stopping=stopping)
    dev = pkg.solve(a, part, cfg)
    monkeypatch.setenv("IBMI_HOST_LOOP", "1")
    host = pkg.solve(a, part, cfg)
    assert dev.iterations == host.iterations and dev.converged == host.converged
    assert dev.error_trace == host.error_trace
    assert dev.power_iterations == host.power_iterations
    assert np.array_equal(dev.result, host.result)
    if stopping == "frobenius":
        np.testing.assert_array_equal(np.isnan(dev.residual_trace), np.isnan(host.residual_trace))
        assert dev.residual_trace[-1] == host.residual_trace[-1] < cfg.tol
    assert len(dev.wall_times) == dev.iterations and all(w > 0 for w in dev.wall_times)
