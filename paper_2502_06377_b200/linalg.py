"""Dense building blocks of the linalg seam on the GPU.

Mirrors the parts of the reference's ``ibmi.linalg`` that the sweep uses
(`/root/reference/pkg/src/ibmi/linalg.py`): ``spd_inverse`` (:122-130),
``two_norm`` (:256-274) and the matrix product (`@`, :175-183), each running
in ``libibmi_b200.so``.  torch is used only to hold device buffers.
"""

from __future__ import annotations

import ctypes as C
import warnings

import numpy as np

from . import _abi
from .device import restart_vector
from .exceptions import DimensionMismatch, NoConvergenceWarning

POWER_RTOL = 1e-9
POWER_MAX_ITERS = 5000
SYMMETRY_RTOL = 1e-12


def _torch():
    import torch

    return torch


def as_matrix(a) -> np.ndarray:
    """linalg.py:52-59 — 2-D nonempty float64."""
    m = np.asarray(a, dtype=np.float64)
    if m.ndim != 2:
        raise DimensionMismatch(f"expected a 2-D matrix, got ndim={m.ndim}")
    if m.shape[0] < 1 or m.shape[1] < 1:
        raise DimensionMismatch(f"matrix must be nonempty, got shape {m.shape}")
    return m


def _to_dev(a, device=0):
    torch = _torch()
    if hasattr(a, "is_cuda") and a.is_cuda:
        return a.to(torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=f"cuda:{device}")


def _stream(t):
    return C.c_void_p(_torch().cuda.current_stream(t.device).cuda_stream)


def spd_inverse(a, device: int = 0):
    """Explicit SPD inverse (linalg.py:122-130): blocked Cholesky, triangular
    inverse and L⁻ᵀL⁻¹ on the device; exactly symmetric output.  Raises
    ``ValueError`` for an asymmetric input and ``NotPositiveDefinite(index)``
    with LAPACK's elimination step for a non-SPD one."""
    host = not (hasattr(a, "is_cuda") and a.is_cuda)
    if host:
        a = as_matrix(a)
        if a.shape[0] != a.shape[1]:
            raise DimensionMismatch(f"expected a square matrix, got shape {a.shape}")
        scale = np.abs(a).max()
        if scale != 0.0 and np.abs(a - a.T).max() > SYMMETRY_RTOL * scale:
            raise ValueError("matrix is not symmetric")
    d = _to_dev(a, device)
    n = d.shape[0]
    out = _torch().empty_like(d)
    piv = C.c_int64(-1)
    rc = _abi.lib().ibmi_spd_inverse(n, C.c_void_p(d.data_ptr()), d.stride(0), C.c_void_p(out.data_ptr()),
                                     out.stride(0), C.byref(piv), _stream(d))
    _abi.check(rc, "spd_inverse", fail_pivot=piv.value)
    return out.cpu().numpy() if host else out


def two_norm(a, rtol: float = POWER_RTOL, max_iters: int = POWER_MAX_ITERS, device: int = 0) -> float:
    """Spectral norm by the reference's power iteration (linalg.py:256-274),
    evaluated in Gram form on the device; warns ``NoConvergenceWarning`` at the cap."""
    host = not (hasattr(a, "is_cuda") and a.is_cuda)
    if host:
        a = as_matrix(a)
    d = _to_dev(a, device)
    rows, cols = d.shape
    if rows < 1 or cols < 1:
        raise DimensionMismatch(f"matrix must be nonempty, got shape {tuple(d.shape)}")
    v = restart_vector(cols)
    s, it, cv = C.c_double(), C.c_int(), C.c_int()
    rc = _abi.lib().ibmi_two_norm(rows, cols, C.c_void_p(d.data_ptr()), d.stride(0), _abi.dbl_ptr(v), float(rtol),
                                  int(max_iters), C.byref(s), C.byref(it), C.byref(cv), _stream(d))
    _abi.check(rc, "two_norm")
    if not cv.value:
        warnings.warn(f"two_norm: power iteration did not stabilize in {max_iters} iterations; "
                      f"returning last estimate {s.value:.6e}", NoConvergenceWarning, stacklevel=2)
    two_norm.last_iterations = it.value
    return s.value


def dgemm_nt(x, y, alpha: float = 1.0, beta: float = 0.0, c=None):
    """``alpha · x · yᵀ + beta · c`` on device tensors through the DMMA GEMM."""
    torch = _torch()
    m, k = x.shape
    n, k2 = y.shape
    if k != k2:
        raise DimensionMismatch(f"inner dimensions differ: {tuple(x.shape)} vs {tuple(y.shape)}")
    if c is None:
        c = torch.zeros((m, n), dtype=torch.float64, device=x.device)
    rc = _abi.lib().ibmi_dgemm_nt(m, n, k, float(alpha), C.c_void_p(x.data_ptr()), x.stride(0),
                                  C.c_void_p(y.data_ptr()), y.stride(0), float(beta), C.c_void_p(c.data_ptr()),
                                  c.stride(0), _stream(x))
    _abi.check(rc, "dgemm_nt")
    return c


def dgemm_nt_ozaki(x, y, moduli: int = 18, alpha: float = 1.0):
    """``alpha · x · yᵀ`` by Ozaki-II emulation on the INT8 tensor cores
    (``ibmi_dgemm_nt_ozaki``): ``moduli`` exact residue GEMMs, CRT, one FP64
    rounding; accurate to 2^-t of each row's largest entry."""
    torch = _torch()
    m, k = x.shape
    n, k2 = y.shape
    if k != k2:
        raise DimensionMismatch(f"inner dimensions differ: {tuple(x.shape)} vs {tuple(y.shape)}")
    c = torch.zeros((m, n), dtype=torch.float64, device=x.device)
    rc = _abi.lib().ibmi_dgemm_nt_ozaki(m, n, k, float(alpha), C.c_void_p(x.data_ptr()), x.stride(0),
                                        C.c_void_p(y.data_ptr()), y.stride(0), C.c_void_p(c.data_ptr()),
                                        c.stride(0), int(moduli), _stream(x))
    _abi.check(rc, "dgemm_nt_ozaki")
    return c


def matmul(a, b):
    """``a @ b`` in float64 (linalg.py:175-183) on the device (a·(bᵀ)ᵀ)."""
    a = as_matrix(a)
    b = as_matrix(b)
    if a.shape[1] != b.shape[0]:
        raise DimensionMismatch(f"inner dimensions differ: {a.shape} @ {b.shape}")
    x = _to_dev(a)
    y = _to_dev(np.ascontiguousarray(b.T))
    return dgemm_nt(x, y).cpu().numpy()
