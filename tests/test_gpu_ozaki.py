"""GPU parity of the Ozaki-II FP64 emulation (INT8 tcgen05 residue GEMMs +
Chinese remaindering, csrc/ozaki.cuh) against long-double products, FP64
DMMA, the oracle and the reference-generated golden fixtures.

The emulated GEMM is exact up to the scaling truncation of each operand row
to t bits (t = min(62, (log2 Π m - 2 - log2 k)/2); 54 at 16 moduli and the c4
panel shape), so its error bound relative to |X|·|Y| sits below FP64 DGEMM's.
The solve-level tests are the DMMA parity tests re-run with every context in
emulation mode (ibmi_tune(7, 16): the default moduli of new contexts), with
the same tolerances: Σ within 1e-10 relative Frobenius of the reference,
error trace within |Δ| <= 1e-6·err_ref + 5e-2·tol, same sweep count.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import random_spd

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

from test_gpu_parity import (  # noqa: E402,F401  (re-collected here, under emulation)
    test_c1_full_solve_matches_reference,
    test_c2_full_solve_frobenius_stop,
    test_c3_full_solve_matches_reference,
    test_c4_through_the_floor_matches_reference,
    test_device_loop_equals_host_loop,
    test_solve_red_black_matches_oracle,
    test_solve_shapes_match_oracle,
    test_solve_small_cases_match_reference,
    test_block_update_and_error_estimate_match_reference,
    test_block_update_noncontiguous_set,
    test_initial_guesses_match_reference,
    test_solve_mixed_runs_and_lists_local_guess,
    test_solve_overlapping_noncontiguous_matches_oracle,
    test_solve_with_guess_matches_oracle,
)

MODULI = 16


@pytest.fixture(scope="module", autouse=True)
def _emulation():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA (run with -m 'not gpu' on CPU hosts)")
    from paper_2502_06377_b200 import _abi

    L = _abi.lib()
    _abi.check(L.ibmi_tune(7, MODULI))
    yield
    _abi.check(L.ibmi_tune(7, 0))


def _ld_ref(x, y):
    ref = x.astype(np.longdouble) @ y.astype(np.longdouble).T
    scale = np.abs(x).astype(np.longdouble) @ np.abs(y).astype(np.longdouble).T
    return ref, scale


def _cases():
    rng = np.random.default_rng(7)
    yield "gauss", rng.standard_normal((256, 1024)), rng.standard_normal((384, 1024))
    yield "row-scaled", rng.standard_normal((200, 700)) * np.exp(rng.uniform(-30, 30, (200, 1))), \
        rng.standard_normal((333, 700)) * np.exp(rng.uniform(-30, 30, (333, 1)))
    yield "entry-scaled", rng.standard_normal((150, 900)) * np.exp(rng.uniform(-6, 6, (150, 900))), \
        rng.standard_normal((170, 900)) * np.exp(rng.uniform(-6, 6, (170, 900)))
    x = rng.standard_normal((130, 257))
    x[3] = 0.0
    x[:, 100] = 0.0
    yield "zeros+odd", x, rng.standard_normal((259, 257))
    yield "tiny", rng.standard_normal((1, 3)), rng.standard_normal((2, 3))


@pytest.mark.parametrize("case", list(range(5)))
def test_ozaki_gemm_accuracy_vs_long_double(case):
    from paper_2502_06377_b200 import linalg

    name, x, y = list(_cases())[case]
    ref, scale = _ld_ref(x, y)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    c_dmma = linalg.dgemm_nt(xd, yd).cpu().numpy()
    e_dmma = float(np.max(np.abs(c_dmma - ref) / np.maximum(scale, 1e-300)))
    for n in (14, 16, 18):
        c = linalg.dgemm_nt_ozaki(xd, yd, n).cpu().numpy()
        e = float(np.max(np.abs(c - ref) / np.maximum(scale, 1e-300)))
        # 16+ moduli: at least as accurate as FP64 DGEMM relative to |X||Y|;
        # 14 moduli (t ~ 50 bits) loses bits on rows with a wide dynamic range
        bound = 1e-12 if n == 14 else max(e_dmma, 1e-15)
        assert e <= bound, (name, n, e, e_dmma)
    assert np.all(c[scale == 0] == 0)


def test_ozaki_gemm_alpha_and_rejects_bad_moduli():
    from paper_2502_06377_b200 import linalg
    from paper_2502_06377_b200.exceptions import DimensionMismatch

    rng = np.random.default_rng(1)
    x = torch.from_numpy(rng.standard_normal((64, 96))).cuda()
    y = torch.from_numpy(rng.standard_normal((80, 96))).cuda()
    c = linalg.dgemm_nt_ozaki(x, y, 16, alpha=-2.5).cpu().numpy()
    ref = -2.5 * (x.cpu().numpy() @ y.cpu().numpy().T)
    assert np.max(np.abs(c - ref)) <= 1e-13 * np.max(np.abs(ref))
    with pytest.raises(ValueError):
        linalg.dgemm_nt_ozaki(x, y, 7)
    with pytest.raises(ValueError):
        linalg.dgemm_nt_ozaki(x, y, 21)
    with pytest.raises(DimensionMismatch):
        linalg.dgemm_nt_ozaki(x, y[:, :50], 16)


def test_emulated_solve_matches_dmma_solve():
    """Same problem, FP64 DMMA vs emulation (per-solve switch IbmiConfig.gemm)."""
    import paper_2502_06377_b200 as pkg

    p = 1536
    a = random_spd(p, 3)
    part = pkg.contiguous_partition(p, 6, 0.125)
    r0 = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-11, gemm="dmma"))
    r1 = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-11, gemm="ozaki", ozaki_moduli=16))
    r2 = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-11, gemm="ozaki", ozaki_moduli=18))
    assert r0.iterations == r1.iterations == r2.iterations
    for r in (r1, r2):
        assert np.linalg.norm(r.result - r0.result) <= 1e-12 * np.linalg.norm(r0.result)
        assert np.array_equal(r.result, r.result.T)
    with pytest.raises(ValueError):
        pkg.IbmiConfig(gemm="ozaki", ozaki_moduli=4)
    with pytest.raises(ValueError):
        pkg.IbmiConfig(gemm="tf32")


def test_emulation_switch_on_context():
    import paper_2502_06377_b200 as pkg
    from paper_2502_06377_b200.device import DeviceSolver

    p = 640
    a = random_spd(p, 5)
    part = pkg.contiguous_partition(p, 3, 0.1)
    with DeviceSolver(a, partition=part) as ds:
        assert ds.emulation == MODULI          # library default set by ibmi_tune(7)
        ds.setup()
        ds.init_sigma(0)
        e_oz = [ds.sweep(1e-9, 5000)[0] for _ in range(4)]
        ds.set_emulation(0)
        assert ds.emulation == 0
        ds.init_sigma(0)
        e_dm = [ds.sweep(1e-9, 5000)[0] for _ in range(4)]
        with pytest.raises(ValueError):
            ds.set_emulation(30)
    assert np.allclose(e_oz, e_dm, rtol=1e-9, atol=0)


@pytest.mark.parametrize("moduli", [16, 18])
def test_residue_planes_overflow_repair(moduli):
    """Σ0 = 1e-6·I: the first Σ_II blocks are ~1e6 times their rows' exponents,
    so the incremental residue planes must flag and re-convert those rows
    (oz_fix_rows_kernel).  Set starts are multiples of 128 (planes path)."""
    import paper_2502_06377_b200 as pkg
    from paper_2502_06377_b200.device import DeviceSolver

    p = 2048
    a = random_spd(p, 11) / p
    part = pkg.contiguous_partition(p, 4, 0.25)
    assert all(s[0] % 128 == 0 for s in part.sets)
    sig0 = 1e-6 * np.eye(p)
    out = {}
    for mode in (0, moduli):
        with DeviceSolver(a, partition=part) as ds:
            ds.set_emulation(mode)
            ds.setup()
            ds.set_sigma(sig0)
            errs = [ds.sweep(1e-9, 5000)[0] for _ in range(4)]
            out[mode] = (errs, ds.sigma())
    e0, s0 = out[0]
    e1, s1 = out[moduli]
    assert np.linalg.norm(s1 - s0) <= 1e-12 * np.linalg.norm(s0)
    assert np.allclose(e1, e0, rtol=1e-9, atol=0)
