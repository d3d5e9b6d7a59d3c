"""Drop-in IBMI solver API on the B200 path.

Names, signatures, defaults, return types and error behaviour follow the
reference's ``ibmi.solver`` (`/root/reference/pkg/src/ibmi/solver.py:41-278`);
every flop runs in ``libibmi_b200.so`` (FP64 DMMA kernels on sm_100a).  There
is no CPU fallback: without the CUDA library these functions raise.

Extensions (all optional, defaults reproduce the reference):

* ``IbmiConfig.initial_guess="jacobi"``: Σ₀[c₁,c₁] = diag(1/A_ii) (BASELINE c1/c2);
* ``IbmiConfig.stopping="frobenius"``: stop on ‖I − AΣ‖_F < tol (BASELINE c2);
* ``SolveReport.power_iterations`` / ``residual_trace`` / ``setup_seconds``;
* ``solve(..., result_on_device=True)`` returns Σ as a CUDA tensor;
* ``IbmiConfig.gemm="ozaki"``: the hot GEMMs run as ``ozaki_moduli`` exact INT8
  tensor-core GEMMs of residues (Ozaki-II FP64 emulation, ``ibmi_set_emulation``)
  instead of FP64 DMMA; ``gemm=None`` keeps the library default (``ibmi_tune(7)``).
"""

from __future__ import annotations

import os
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .device import DeviceSolver
from .exceptions import DeviceError, DimensionMismatch, NoConvergenceWarning
from .partition import Partition, complement, validate

__all__ = [
    "GUESS_CHOICES",
    "IbmiConfig",
    "SolveReport",
    "block_update",
    "error_estimate",
    "initial_guess_identity",
    "initial_guess_local_inverse",
    "initial_guess_monte_carlo",
    "initial_guess_takahashi",
    "make_initial_guess",
    "run_solve",
    "solve",
]

POWER_RTOL = 1e-9          # reference linalg.py:47
POWER_MAX_ITERS = 5000     # reference linalg.py:48

GUESS_IDENTITY = "identity"
GUESS_LOCAL_INVERSE = "local"
GUESS_MONTE_CARLO = "mc"
GUESS_TAKAHASHI = "takahashi"
GUESS_JACOBI = "jacobi"
GUESS_CHOICES = (GUESS_IDENTITY, GUESS_LOCAL_INVERSE, GUESS_MONTE_CARLO, GUESS_TAKAHASHI, GUESS_JACOBI)
STOPPING_CHOICES = ("estimate", "frobenius")
GEMM_CHOICES = (None, "dmma", "ozaki")


@dataclass(frozen=True)
class IbmiConfig:
    """Solver controls (reference solver.py:62-91, same fields and checks)."""

    tol: float = 1e-8
    max_iterations: int = 500
    initial_guess: str = GUESS_IDENTITY
    mc_samples: int = 100
    mc_seed: int = 0
    norm_rtol: float = POWER_RTOL
    norm_max_iters: int = POWER_MAX_ITERS
    stopping: str = "estimate"
    residual_every_sweep: bool = False
    gemm: str | None = None
    ozaki_moduli: int = 16

    def __post_init__(self):
        if not self.tol > 0:
            raise ValueError(f"tol must be positive, got {self.tol}")
        if self.max_iterations < 1:
            raise ValueError(f"max_iterations must be >= 1, got {self.max_iterations}")
        if self.initial_guess not in GUESS_CHOICES:
            raise ValueError(
                f"unknown initial guess {self.initial_guess!r}; expected one of {GUESS_CHOICES}")
        if self.initial_guess == GUESS_MONTE_CARLO and self.mc_samples < 1:
            raise ValueError(f"mc_samples must be >= 1, got {self.mc_samples}")
        if self.stopping not in STOPPING_CHOICES:
            raise ValueError(f"unknown stopping rule {self.stopping!r}; expected one of {STOPPING_CHOICES}")
        if self.gemm not in GEMM_CHOICES:
            raise ValueError(f"unknown gemm {self.gemm!r}; expected one of {GEMM_CHOICES}")
        if self.gemm == "ozaki" and not 8 <= self.ozaki_moduli <= 20:
            raise ValueError(f"ozaki_moduli must be in [8, 20], got {self.ozaki_moduli}")


@dataclass
class SolveReport:
    """Outcome of one solve (reference solver.py:94-106) plus device extras."""

    iterations: int
    converged: bool
    error_trace: list[float]
    wall_times: list[float]
    result: object = field(repr=False)
    power_iterations: list[int] = field(default_factory=list)
    residual_trace: list[float] = field(default_factory=list)
    setup_seconds: float = 0.0

    @property
    def total_seconds(self) -> float:
        return float(sum(self.wall_times))


def initial_guess_identity(comp_size: int) -> np.ndarray:
    """solver.py:158-159."""
    return np.eye(comp_size)


def initial_guess_local_inverse(a, comp) -> np.ndarray:
    """solver.py:162-164 — inverse of A[c, c], computed on the GPU."""
    from .linalg import spd_inverse

    comp = np.asarray(comp, dtype=np.intp)
    a = np.asarray(a, dtype=np.float64)
    return spd_inverse(a[np.ix_(comp, comp)])


def _mc_draws(p: int, n_samples: int, seed: int) -> np.ndarray:
    """The reference's standard-normal draws (solver.py:178), so the GPU guess
    matches it sample for sample."""
    return np.random.default_rng(seed).standard_normal((p, n_samples))


def initial_guess_monte_carlo(a, comp, n_samples: int, seed: int) -> np.ndarray:
    """solver.py:167-181 — sample covariance of L⁻ᵀw on ``comp``; Cholesky,
    triangular inverse and both products on the GPU (``ibmi_mc_guess``)."""
    import ctypes as C

    import torch

    if n_samples < 1:
        raise ValueError(f"n_samples must be >= 1, got {n_samples}")
    comp = np.ascontiguousarray(np.asarray(comp, dtype=np.int64))
    if hasattr(a, "is_cuda") and a.is_cuda:
        da = a.to(torch.float64).contiguous()
    else:
        da = torch.as_tensor(np.ascontiguousarray(np.asarray(a, dtype=np.float64)), device="cuda")
    p = da.shape[0]
    w = np.ascontiguousarray(_mc_draws(p, n_samples, seed))
    out = torch.zeros((comp.size, comp.size), dtype=torch.float64, device="cuda")
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _abi.check(_abi.lib().ibmi_mc_guess(p, C.c_void_p(da.data_ptr()), da.stride(0), C.c_void_p(w.ctypes.data), n_samples,
                                        C.c_void_p(comp.ctypes.data), comp.size, C.c_void_p(out.data_ptr()),
                                        comp.size, st), "mc_guess")
    return out.cpu().numpy()


def initial_guess_takahashi(a, comp) -> np.ndarray:
    """solver.py:184-212 — the comp × comp block of A⁻¹, which the reference's
    LDLᵀ backward recurrence reproduces; on the GPU it is S_c⁻¹ with
    S_c = A_cc − A_cI A_II⁻¹ A_Ic (``IBMI_GUESS_TAKAHASHI``)."""
    a = np.asarray(a, dtype=np.float64)
    comp = np.asarray(comp, dtype=np.int64)
    p = a.shape[0]
    keep = np.ones(p, dtype=bool)
    keep[comp] = False
    rest = np.nonzero(keep)[0]
    perm = np.concatenate([rest, comp])
    with DeviceSolver(a, [(0, rest.size), (rest.size, p)], perm=perm) as ds:
        ds.setup(0, 1)
        ds.init_sigma(_abi.GUESS_TAKAHASHI)
        s = ds.sigma()
    return s[np.ix_(comp, comp)]


def make_initial_guess(a, comp, cfg: IbmiConfig) -> np.ndarray:
    """solver.py:215-222 (plus the BASELINE ``jacobi`` seed), all on the GPU."""
    if cfg.initial_guess == GUESS_IDENTITY:
        return initial_guess_identity(len(comp))
    if cfg.initial_guess == GUESS_LOCAL_INVERSE:
        return initial_guess_local_inverse(a, comp)
    if cfg.initial_guess == GUESS_MONTE_CARLO:
        return initial_guess_monte_carlo(a, comp, cfg.mc_samples, cfg.mc_seed)
    if cfg.initial_guess == GUESS_JACOBI:
        d = np.diag(np.asarray(a, dtype=np.float64))[np.asarray(comp, dtype=np.intp)]
        return np.diag(1.0 / d)
    return initial_guess_takahashi(a, comp)


_GUESS_KIND = {GUESS_IDENTITY: _abi.GUESS_IDENTITY, GUESS_JACOBI: _abi.GUESS_JACOBI,
               GUESS_LOCAL_INVERSE: _abi.GUESS_LOCAL, GUESS_TAKAHASHI: _abi.GUESS_TAKAHASHI,
               GUESS_MONTE_CARLO: _abi.GUESS_MC}


def _shape_of(a):
    return tuple(a.shape) if hasattr(a, "shape") else np.asarray(a).shape


def solve(a, part: Partition, cfg: IbmiConfig | None = None, *, device: int = 0,
          result_on_device: bool = False, callback=None) -> SolveReport:
    """Approximate ``inv(A)`` by sweeping block updates over ``part``
    (reference solver.py:225-278).

    Each sweep applies the sets' updates in order, then evaluates the
    reference's error estimate on the last set; the solve stops when it is
    ≤ ``cfg.tol`` (or ‖I − AΣ‖_F < tol with ``stopping="frobenius"``).
    Hitting ``max_iterations`` gives ``converged=False``; it is not raised.
    ``a`` may be a numpy array or a float64 CUDA tensor already in HBM.
    """
    cfg = cfg or IbmiConfig()
    stopping = getattr(cfg, "stopping", "estimate")      # reference IbmiConfig has no such field
    if not hasattr(a, "is_cuda"):
        a = np.asarray(a, dtype=np.float64)
    validate(part)
    if _shape_of(a) != (part.p, part.p):
        raise DimensionMismatch(
            f"matrix shape {_shape_of(a)} does not match partition over {part.p} indices")
    if cfg.initial_guess not in _GUESS_KIND:
        raise NotImplementedError(f"initial guess {cfg.initial_guess!r} is not available on the B200 path yet")

    prof = os.environ.get("IBMI_PROFILE") is not None
    t0 = time.perf_counter()
    ds = DeviceSolver(a, partition=part, device=device)
    t1 = time.perf_counter()
    try:
        return run_solve(ds, part, cfg, a=a, result_on_device=result_on_device, callback=callback)
    finally:
        t2 = time.perf_counter()
        ds.close()
        if prof:
            import sys

            print(f"[ibmi] context + A upload {t1 - t0:.3f}s, solve {t2 - t1:.3f}s, release {time.perf_counter() - t2:.3f}s",
                  file=sys.stderr)


def run_solve(ds: DeviceSolver, part: Partition, cfg: IbmiConfig, *, a=None, result_on_device: bool = False,
              callback=None, fetch_result: bool = True) -> SolveReport:
    """The sweep loop of ``solve`` (solver.py:241-278) on a prepared device state."""
    prof = os.environ.get("IBMI_PROFILE") is not None
    stopping = getattr(cfg, "stopping", "estimate")
    gemm = getattr(cfg, "gemm", None)
    if gemm is not None:
        ds.set_emulation(int(getattr(cfg, "ozaki_moduli", 16)) if gemm == "ozaki" else 0)
    t0 = time.perf_counter()
    ds.setup()
    kind = _GUESS_KIND[cfg.initial_guess]
    if kind == _abi.GUESS_MC:
        if ds.perm is None:
            ds.init_sigma(kind, _mc_draws(part.p, cfg.mc_samples, cfg.mc_seed))
        else:   # relabelled partition: draw in the original order, insert the block
            comp0 = complement(part, 0)
            ds.init_sigma(_abi.GUESS_MATRIX, initial_guess_monte_carlo(a, comp0, cfg.mc_samples, cfg.mc_seed))
    else:
        ds.init_sigma(kind)
    setup_s = time.perf_counter() - t0
    if callback is None and os.environ.get("IBMI_HOST_LOOP") is None:
        try:
            r = ds.solve_loop(cfg.tol, cfg.max_iterations, cfg.norm_rtol, cfg.norm_max_iters, stopping,
                             cfg.residual_every_sweep)
        except (NotImplementedError, DeviceError):
            r = None            # conditional graphs unavailable: host-driven loop below
        if r is not None:
            for ok in r["power_conv"]:
                if not ok:
                    warnings.warn(f"two_norm: power iteration did not stabilize in {cfg.norm_max_iters} "
                                  "iterations; returning last estimate", NoConvergenceWarning, stacklevel=3)
            t1 = time.perf_counter()
            result = ds.sigma(on_device=result_on_device) if fetch_result else None
            if prof:
                import sys

                print(f"[ibmi] setup {setup_s:.3f}s device loop {sum(r['sweep_seconds']):.3f}s "
                      f"download {time.perf_counter() - t1:.3f}s", file=sys.stderr)
            return SolveReport(iterations=r["sweeps"], converged=r["converged"], error_trace=r["error_trace"],
                               wall_times=r["sweep_seconds"], result=result, power_iterations=r["power_iters"],
                               residual_trace=r["residual_trace"], setup_seconds=setup_s)
    errs, walls, pits, resid = [], [], [], []
    converged, it = False, 0
    while it < cfg.max_iterations:
        start = time.perf_counter()
        it += 1
        err, pit, pconv = ds.sweep(cfg.norm_rtol, cfg.norm_max_iters)
        # ‖I − AΣ‖_F ≥ ‖(ΣA)_Ic‖_F = ‖B‖_F ≥ ‖B‖₂ ≥ err (the power iteration approaches ‖B‖₂
        # from below), so while err ≥ tol (with a rounding margin) the residual cannot be
        # < tol and its 2p³ evaluation is skipped without changing the stopping sweep.
        fr = None
        if stopping == "frobenius":
            if getattr(cfg, "residual_every_sweep", False) or err < 1.01 * cfg.tol:
                fr = ds.frobenius()
            else:
                fr = float("nan")
        walls.append(time.perf_counter() - start)
        if not pconv:
            warnings.warn(
                f"two_norm: power iteration did not stabilize in {cfg.norm_max_iters} "
                f"iterations; returning last estimate {err:.6e}", NoConvergenceWarning, stacklevel=3)
        errs.append(err)
        pits.append(pit)
        if fr is not None:
            resid.append(fr)
        if callback is not None:
            callback(it, err, fr)
        if (fr < cfg.tol) if fr is not None else (err <= cfg.tol):   # nan < tol is False
            converged = True
            break
    t1 = time.perf_counter()
    result = ds.sigma(on_device=result_on_device) if fetch_result else None
    if prof:
        import sys

        print(f"[ibmi] setup {setup_s:.3f}s sweeps {sum(walls):.3f}s download {time.perf_counter() - t1:.3f}s",
              file=sys.stderr)
    return SolveReport(iterations=it, converged=converged, error_trace=errs, wall_times=walls, result=result,
                       power_iterations=pits, residual_trace=resid, setup_seconds=setup_s)


def _single_set(a, sigma, idx, comp):
    """Shared argument handling of block_update / error_estimate: returns the
    device layout (ranges or a relabelling putting idx first)."""
    p = sigma.shape[0]
    idx = np.asarray(idx, dtype=np.intp).ravel()
    comp = np.asarray(comp, dtype=np.intp).ravel()
    allidx = np.concatenate([idx, comp])
    if idx.size == 0 or allidx.size != p or not np.array_equal(np.sort(allidx), np.arange(p)):
        raise ValueError("idx and comp must partition every row/column index")
    if np.array_equal(idx, np.arange(idx[0], idx[0] + idx.size)) and \
            np.array_equal(comp, np.concatenate([np.arange(0, idx[0]), np.arange(idx[-1] + 1, p)])):
        return [(int(idx[0]), int(idx[-1]) + 1)], None
    # relabel: idx first (in the given order), then comp in the given order
    return [(0, idx.size)], np.concatenate([idx, comp]).astype(np.int64)


def _is_symmetric(sigma: np.ndarray) -> bool:
    return sigma.size == 0 or bool(np.array_equal(sigma, sigma.T))


def _export(ds: DeviceSolver, which: int, k: int = 0):
    import ctypes as C

    ptr, r, c, ld = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int64()
    _abi.check(_abi.lib().ibmi_export(ds._h, which, k, C.byref(ptr), C.byref(r), C.byref(c), C.byref(ld)), "export")
    return ptr.value, ld.value


def _diag_block_nonsymmetric(ds: DeviceSolver) -> None:
    """Σ_II = A_II⁻¹ + ½(M Wᵀ + W Mᵀ) after K1 has stored Σ[I, c] = −M.

    solver.py:125-127 symmetrises ``ainv + M Wᵀ``; with a symmetric Σ the
    library's K2 takes the lower triangle of ``M Wᵀ`` (symmetric up to
    rounding), but with a non-symmetric Σ_cc that product is not symmetric,
    so the average is formed by two GEMMs on the device:
    ``Σ_II = ainv + ½·M Wᵀ`` then ``Σ_II += ½·W Mᵀ``."""
    import ctypes as C

    lo, hi = ds.ranges[0]
    p, b = ds.p, hi - lo
    s_ptr, lds = _export(ds, 1)
    w_ptr, ldw = _export(ds, 2, 0)
    ai_ptr, ldai = _export(ds, 3, 0)
    run = _abi.Map.run
    for x, ldx, xm, y, ldy, yn, d, ldd, dm in (
            (s_ptr, lds, run(lo), w_ptr, ldw, run(0), ai_ptr, ldai, run(0)),     # ainv − ½(−M)Wᵀ
            (w_ptr, ldw, run(0), s_ptr, lds, run(lo), s_ptr, lds, run(lo))):     # + (−½)·W(−M)ᵀ
        g = _abi.GemmDesc()
        g.x, g.ldx, g.xm, g.xrows, g.xcols = x, ldx, xm, 0, 0
        g.y, g.ldy, g.yn, g.yrows, g.ycols = y, ldy, yn, 0, 0
        g.m, g.n = b, b
        segs = [(0, 0, lo), (hi, hi, p - hi)]
        segs = [sg for sg in segs if sg[2] > 0]
        g.nseg = len(segs)
        for i, (x0, y0, ln) in enumerate(segs):
            g.seg_x0[i], g.seg_y0[i], g.seg_len[i] = x0, y0, ln
        g.c, g.ldc, g.cm, g.cn, g.direct = s_ptr, lds, run(lo), run(lo), 1
        g.alpha, g.beta, g.d, g.ldd, g.dm, g.dn = -0.5, 1.0, d, ldd, dm, run(0) if d == ai_ptr else run(lo)
        g.splits = 1
        _abi.check(_abi.lib().ibmi_gemm(C.byref(g), C.c_void_p(ds.stream_handle())), "gemm")


def block_update(a, sigma, idx, comp) -> None:
    """Apply one block-inverse update to ``sigma`` in place (solver.py:132-144).

    Like the reference, only a float64 ndarray ``sigma`` is updated in place;
    any other input is converted and the result is discarded.  ``sigma`` need
    not be symmetric: the kernels read Σ[c, c] through rows of the device
    copy, so a non-symmetric Σ is uploaded as Σᵀ.  The update writes only
    mirrored pairs (Σ_Ic = −M, Σ_cI = −Mᵀ, a symmetric Σ_II) and leaves
    Σ[c, c] untouched, so transposing back gives the reference's result; Σ_II
    is then the average ``ainv + ½(M Wᵀ + W Mᵀ)`` (:func:`_diag_block_nonsymmetric`).
    """
    a = np.asarray(a, dtype=np.float64)
    sigma = np.asarray(sigma)
    if a.shape != sigma.shape or a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionMismatch(f"matrix/approximation shapes differ: {a.shape} vs {sigma.shape}")
    target = sigma if sigma.dtype == np.float64 else np.asarray(sigma, dtype=np.float64)
    ranges, perm = _single_set(a, target, idx, comp)
    sym = _is_symmetric(target)
    with DeviceSolver(a, ranges, perm=perm) as ds:
        ds.setup()
        ds.set_sigma(target if sym else target.T)
        ds.block_update(0)
        if not sym:
            _diag_block_nonsymmetric(ds)
        out = ds.sigma()
    target[...] = out if sym else out.T


def error_estimate(a, sigma, idx, comp, rtol: float = POWER_RTOL, max_iters: int = POWER_MAX_ITERS) -> float:
    """Spectral norm of ``S_I A_{I,c} + S_{I,c} A_c`` (solver.py:147-155), any float64 Σ."""
    a = np.asarray(a, dtype=np.float64)
    sigma = np.asarray(sigma, dtype=np.float64)
    if a.shape != sigma.shape or a.ndim != 2 or a.shape[0] != a.shape[1]:
        raise DimensionMismatch(f"matrix/approximation shapes differ: {a.shape} vs {sigma.shape}")
    # B = Σ[I, :]·A[:, c] reads rows of Σ, so any (also non-symmetric) Σ is used as given
    ranges, perm = _single_set(a, sigma, idx, comp)
    if ranges[0][1] - ranges[0][0] == a.shape[0]:
        raise DimensionMismatch("matrix must be nonempty, got shape (%d, 0)" % a.shape[0])
    with DeviceSolver(a, ranges, perm=perm) as ds:
        ds.set_sigma(sigma)
        err, _, conv = ds.error_estimate(0, rtol, max_iters)
    if not conv:
        warnings.warn(f"two_norm: power iteration did not stabilize in {max_iters} iterations; "
                      f"returning last estimate {err:.6e}", NoConvergenceWarning, stacklevel=2)
    return err
