"""Dense building blocks of the linalg seam on the GPU.

Mirrors the reference's ``ibmi.linalg`` seam, "the only place that talks to
LAPACK/BLAS" (`/root/reference/pkg/src/ibmi/linalg.py:1-8`):
``cholesky`` / ``chol_solve`` / ``CholeskyFactor`` (:80-119), ``spd_inverse``
(:122-130), ``matmul`` (:175-183), ``gather`` / ``scatter_add_assign``
(:186-211) and ``two_norm`` (:256-274), each running in ``libibmi_b200.so``.
Same argument checks and exception classes as the reference; host (numpy)
inputs give host results, CUDA tensors stay on the device.  torch is used only
to hold device buffers.
"""

from __future__ import annotations

import ctypes as C
import warnings
from dataclasses import dataclass

import numpy as np

from . import _abi
from .device import restart_vector
from .exceptions import DimensionMismatch, IndexOutOfRange, NoConvergenceWarning

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


def _is_dev(a) -> bool:
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def _require_square(a) -> None:
    if a.shape[0] != a.shape[1]:
        raise DimensionMismatch(f"expected a square matrix, got shape {tuple(a.shape)}")


def _require_symmetric(a, rtol: float = SYMMETRY_RTOL) -> None:
    """linalg.py:68-77 — max|a − aᵀ| ≤ rtol · max|a| (device tensors checked on the device)."""
    if _is_dev(a):
        scale = float(a.abs().max())
        skew = float((a - a.T).abs().max()) if scale != 0.0 else 0.0
    else:
        scale = float(np.abs(a).max())
        skew = float(np.abs(a - a.T).max()) if scale != 0.0 else 0.0
    if scale != 0.0 and skew > rtol * scale:
        raise ValueError(f"matrix is not symmetric: max |a - a.T| = {skew:.3e} "
                         f"exceeds {rtol:.1e} * max|a| = {rtol * scale:.3e}")


def _as_dev_matrix(a, device=0):
    """2-D nonempty float64 operand on the device (host arrays are uploaded)."""
    if _is_dev(a):
        if a.ndim != 2:
            raise DimensionMismatch(f"expected a 2-D matrix, got ndim={a.ndim}")
        if a.shape[0] < 1 or a.shape[1] < 1:
            raise DimensionMismatch(f"matrix must be nonempty, got shape {tuple(a.shape)}")
        return _to_dev(a, device), False
    return _to_dev(as_matrix(a), device), True


@dataclass(frozen=True)
class CholeskyFactor:
    """Lower-triangular factor ``l`` with ``l @ l.T`` equal to the input (linalg.py:80-85).
    ``l`` is a numpy array for host inputs and a CUDA tensor for device inputs."""

    l: object
    dim: int


def cholesky(a, device: int = 0) -> CholeskyFactor:
    """Factor an SPD matrix as ``l @ l.T`` (linalg.py:96-109) with the blocked
    device Cholesky; the strict upper triangle of ``l`` is zero.  Raises
    ``NotPositiveDefinite(index)`` with LAPACK's failing elimination step."""
    d, host = _as_dev_matrix(a, device)
    _require_square(d)
    _require_symmetric(d)
    n = d.shape[0]
    out = _torch().empty_like(d)
    piv = C.c_int64(-1)
    rc = _abi.lib().ibmi_cholesky(n, C.c_void_p(d.data_ptr()), d.stride(0), C.c_void_p(out.data_ptr()),
                                  out.stride(0), C.byref(piv), _stream(d))
    _abi.check(rc, "cholesky", fail_pivot=piv.value)
    return CholeskyFactor(l=out.cpu().numpy() if host else out, dim=n)


def chol_solve(f: CholeskyFactor, b, device: int = 0):
    """Solve ``(l @ l.T) @ x = b`` (linalg.py:112-119) on the device."""
    bd, host = _as_dev_matrix(b, device)
    if bd.shape[0] != f.dim:
        raise DimensionMismatch(f"factor dimension {f.dim} does not match rhs rows {bd.shape[0]}")
    ld = _to_dev(f.l, bd.device.index)
    x = _torch().empty_like(bd)
    rc = _abi.lib().ibmi_chol_solve(f.dim, C.c_void_p(ld.data_ptr()), ld.stride(0), bd.shape[1],
                                    C.c_void_p(bd.data_ptr()), bd.stride(0), C.c_void_p(x.data_ptr()), x.stride(0),
                                    _stream(bd))
    _abi.check(rc, "chol_solve")
    return x.cpu().numpy() if host else x


def _check_indices(idx, bound: int, what: str) -> np.ndarray:
    """linalg.py:214-220."""
    if _is_dev(idx):
        idx = idx.cpu().numpy()
    idx = np.asarray(idx, dtype=np.intp)
    if idx.ndim != 1:
        raise DimensionMismatch(f"{what} index list must be 1-D")
    if idx.size and (idx.min() < 0 or idx.max() >= bound):
        raise IndexOutOfRange(f"{what} index out of range [0, {bound})")
    return idx


def _index_tensor(idx: np.ndarray, dev):
    return _torch().as_tensor(np.ascontiguousarray(idx, dtype=np.int64), device=dev)


def gather(a, rows, cols, device: int = 0):
    """``a[rows[i], cols[j]]`` as a fresh matrix (linalg.py:186-191), copied by
    the device gather kernel."""
    d, host = _as_dev_matrix(a, device)
    rows = _check_indices(rows, d.shape[0], "row")
    cols = _check_indices(cols, d.shape[1], "column")
    out = _torch().empty((rows.size, cols.size), dtype=_torch().float64, device=d.device)
    if rows.size and cols.size:
        rt, ct = _index_tensor(rows, d.device), _index_tensor(cols, d.device)
        rc = _abi.lib().ibmi_gather(C.c_void_p(d.data_ptr()), d.stride(0), C.c_void_p(rt.data_ptr()), rows.size,
                                    C.c_void_p(ct.data_ptr()), cols.size, C.c_void_p(out.data_ptr()),
                                    max(out.stride(0), 1), _stream(d))
        _abi.check(rc, "gather")
    return out.cpu().numpy() if host else out


def _last_occurrence(idx: np.ndarray):
    """Unique indices of ``idx`` with the position of their last occurrence:
    NumPy's fancy assignment keeps the last of repeated writes."""
    rev = idx[::-1]
    uniq, first_in_rev = np.unique(rev, return_index=True)
    return uniq, idx.size - 1 - first_in_rev


def scatter_add_assign(target, rows, cols, src, add: bool = False, device: int = 0) -> None:
    """Write ``src`` into ``target`` at the grid ``rows × cols`` (linalg.py:194-211);
    ``add=True`` accumulates.  Like the reference, a float64 ndarray (or CUDA
    tensor) target is updated in place; any other target is converted and the
    result discarded."""
    torch = _torch()
    if _is_dev(target):
        t = target
        if t.dtype != torch.float64 or t.stride(1) != 1:
            t = t.to(torch.float64).contiguous()
        host_target = None
    else:
        host_target = as_matrix(target)
        t = _to_dev(host_target, device)
    s = _to_dev(src, t.device.index) if _is_dev(src) else _to_dev(as_matrix(src), t.device.index)
    if s.ndim != 2 or s.shape[0] < 1 or s.shape[1] < 1:
        raise DimensionMismatch(f"matrix must be nonempty, got shape {tuple(s.shape)}")
    rows = _check_indices(rows, t.shape[0], "row")
    cols = _check_indices(cols, t.shape[1], "column")
    if tuple(s.shape) != (len(rows), len(cols)):
        raise DimensionMismatch(f"source shape {tuple(s.shape)} does not match index grid "
                                f"({len(rows)}, {len(cols)})")
    ur, pr = _last_occurrence(rows)
    uc, pc = _last_occurrence(cols)
    if ur.size != rows.size or uc.size != cols.size:
        s = s.index_select(0, _index_tensor(pr, t.device)).index_select(1, _index_tensor(pc, t.device)).contiguous()
        rows, cols = ur, uc
    rt, ct = _index_tensor(rows, t.device), _index_tensor(cols, t.device)
    rc = _abi.lib().ibmi_scatter(C.c_void_p(t.data_ptr()), t.stride(0), C.c_void_p(rt.data_ptr()), rows.size,
                                 C.c_void_p(ct.data_ptr()), cols.size, C.c_void_p(s.data_ptr()), s.stride(0),
                                 int(bool(add)), _stream(t))
    _abi.check(rc, "scatter_add_assign")
    if host_target is not None:
        host_target[...] = t.cpu().numpy()
    elif t is not target:
        target.copy_(t)


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
