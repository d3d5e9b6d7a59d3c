"""ctypes binding of ``libibmi_b200.so`` (declared in ``include/ibmi_b200.h``).

There is no CPU fallback: if the shared library is missing or cannot be
loaded, :func:`lib` raises.  Status codes become the reference's exception
classes (`/root/reference/pkg/src/ibmi/exceptions.py`) via :func:`check`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .exceptions import (DeviceError, DimensionMismatch, IndexOutOfRange, IoError, NotPositiveDefinite,
                         OutOfMemoryBudget)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libibmi_b200.so")

(OK, ERR_INVALID, ERR_DIM, ERR_INDEX, ERR_NOT_SPD, ERR_NOT_SYMMETRIC, ERR_CUDA, ERR_OOM, ERR_STATE, ERR_UNSUPPORTED,
 ERR_IO) = range(11)
GUESS_IDENTITY, GUESS_JACOBI, GUESS_MATRIX, GUESS_LOCAL, GUESS_MC, GUESS_TAKAHASHI = range(6)

# (name, restype, argtypes) — the full exported surface of include/ibmi_b200.h
_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I64 = C.c_int64
SIGNATURES = [
    ("ibmi_last_error", C.c_char_p, []),
    ("ibmi_version", C.c_char_p, []),
    ("ibmi_create", C.c_int, [C.POINTER(_P), C.c_int, _I64, _P]),
    ("ibmi_destroy", C.c_int, [_P]),
    ("ibmi_set_matrix", C.c_int, [_P, _P, _I64, C.c_int]),
    ("ibmi_load_ibmi1", C.c_int, [_P, C.c_char_p]),
    ("ibmi_save_sigma_ibmi1", C.c_int, [_P, C.c_char_p]),
    ("ibmi_set_partition", C.c_int, [_P, C.c_int, C.POINTER(_I64), C.POINTER(_I64)]),
    ("ibmi_set_partition_general", C.c_int, [_P, C.c_int, C.POINTER(_I64), C.POINTER(_I64)]),
    ("ibmi_setup", C.c_int, [_P, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(_I64)]),
    ("ibmi_init_sigma", C.c_int, [_P, C.c_int, _P, _I64, C.c_int]),
    ("ibmi_set_sigma", C.c_int, [_P, _P, _I64, C.c_int]),
    ("ibmi_get_sigma", C.c_int, [_P, _P, _I64, C.c_int]),
    ("ibmi_copy_rows", C.c_int, [C.c_int, _P, _I64, _P, _I64, _I64, _I64, _P, C.c_int, _P]),
    ("ibmi_set_restart_vector", C.c_int, [_P, _I64, _D]),
    ("ibmi_block_update", C.c_int, [_P, C.c_int]),
    ("ibmi_error_estimate", C.c_int, [_P, C.c_int, C.c_double, C.c_int, _D, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("ibmi_sweep", C.c_int, [_P, C.c_double, C.c_int, _D, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("ibmi_sweep_timed", C.c_int, [_P, C.c_double, C.c_int, _D, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                   C.POINTER(C.c_float)]),
    ("ibmi_solve_loop", C.c_int, [_P, C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, C.POINTER(C.c_int),
                                  C.POINTER(C.c_int), _D, C.POINTER(C.c_int), C.POINTER(C.c_int), _D, _D]),
    ("ibmi_frobenius_residual", C.c_int, [_P, _D]),
    ("ibmi_device_bytes", C.c_int, [_P, C.POINTER(_I64)]),
    ("ibmi_dgemm_nt", C.c_int, [_I64, _I64, _I64, C.c_double, _P, _I64, _P, _I64, C.c_double, _P, _I64, _P]),
    ("ibmi_set_emulation", C.c_int, [_P, C.c_int]),
    ("ibmi_emulation_timing", C.c_int, [_P, _P, _P]),
    ("ibmi_get_emulation", C.c_int, [_P, _P]),
    ("ibmi_dgemm_nt_ozaki", C.c_int, [_I64, _I64, _I64, C.c_double, _P, _I64, _P, _I64, _P, _I64, C.c_int, _P]),
    ("ibmi_spd_inverse", C.c_int, [_I64, _P, _I64, _P, _I64, C.POINTER(_I64), _P]),
    ("ibmi_cholesky", C.c_int, [_I64, _P, _I64, _P, _I64, C.POINTER(_I64), _P]),
    ("ibmi_chol_solve", C.c_int, [_I64, _P, _I64, _I64, _P, _I64, _P, _I64, _P]),
    ("ibmi_gather", C.c_int, [_P, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
    ("ibmi_scatter", C.c_int, [_P, _I64, _P, _I64, _P, _I64, _P, _I64, C.c_int, _P]),
    ("ibmi_sym_rows", C.c_int, [_P, _I64, _P, _I64, _P, _I64, _I64, _P, _I64, _P]),
    ("ibmi_mc_guess", C.c_int, [_I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
    ("ibmi_two_norm", C.c_int, [_I64, _I64, _P, _I64, _D, C.c_double, C.c_int, _D, C.POINTER(C.c_int),
                                C.POINTER(C.c_int), _P]),
    ("ibmi_two_norm_gram", C.c_int, [_I64, _I64, _P, _I64, _P, _I64, _P, _D, C.c_double, C.c_int, _D,
                                     C.POINTER(C.c_int), C.POINTER(C.c_int), _P]),
    ("ibmi_gemm", C.c_int, [_P, _P]),
    ("ibmi_gemm_workspace", C.c_int, [_P, C.POINTER(_I64)]),
    ("ibmi_context_stream", C.c_int, [_P, C.POINTER(_P)]),
    ("ibmi_export", C.c_int, [_P, C.c_int, C.c_int, C.POINTER(_P), C.POINTER(_I64), C.POINTER(_I64),
                              C.POINTER(_I64)]),
    ("ibmi_device_alloc", C.c_int, [C.c_int, _I64, C.POINTER(_P)]),
    ("ibmi_device_free", C.c_int, [_P]),
    ("ibmi_ipc_handle", C.c_int, [_P, C.c_char_p]),
    ("ibmi_ipc_open", C.c_int, [C.c_int, C.c_char_p, C.POINTER(_P)]),
    ("ibmi_ipc_close", C.c_int, [_P]),
    ("ibmi_release_cached_memory", C.c_int, [C.c_int]),
    ("ibmi_cached_bytes", C.c_int, [C.c_int, C.POINTER(_I64)]),
    ("ibmi_launch_count", C.c_longlong, []),
    ("ibmi_tune", C.c_int, [C.c_int, C.c_int]),
    ("ibmi_probe_fp64_peak", C.c_int, [C.c_int, _D]),
]

_lock = threading.Lock()
_lib = None


def lib():
    """Load (once) and return the CUDA library; raise if it is unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2502_06377_b200.build` "
                    "(there is no CPU fallback)")
            h = C.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                f = getattr(h, name)
                f.restype = res
                f.argtypes = args
            _lib = h
    return _lib


def last_error() -> str:
    return lib().ibmi_last_error().decode(errors="replace")


def check(rc: int, what: str = "", *, fail_set: int | None = None, fail_pivot: int | None = None) -> None:
    """Raise the reference's exception class for a non-zero status."""
    if rc == OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == ERR_NOT_SPD:
        raise NotPositiveDefinite(int(fail_pivot if fail_pivot is not None else -1),
                                  f"non-positive pivot at elimination step {fail_pivot}"
                                  + (f" (set {fail_set})" if fail_set is not None and fail_set >= 0 else ""),
                                  set_index=fail_set)
    if rc in (ERR_INVALID, ERR_NOT_SYMMETRIC, ERR_STATE):
        raise ValueError(msg)
    if rc == ERR_DIM:
        raise DimensionMismatch(msg)
    if rc == ERR_INDEX:
        raise IndexOutOfRange(msg)
    if rc == ERR_OOM:
        raise OutOfMemoryBudget(msg)
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == ERR_IO:
        raise IoError(msg)
    raise DeviceError(msg)


def dptr(arr) -> int:
    """Raw address of a numpy array or a CUDA tensor (``data_ptr``)."""
    if isinstance(arr, np.ndarray):
        return arr.ctypes.data
    return int(arr.data_ptr())


def dbl_ptr(arr: np.ndarray):
    return arr.ctypes.data_as(_D)


RUN = 2 ** 62   # "no gap" split value of an ibmi_map


class Map(C.Structure):
    """``ibmi_map``: logical i -> i < split ? off0 + i : off1 + (i - split)."""
    _fields_ = [("split", C.c_int64), ("off0", C.c_int64), ("off1", C.c_int64), ("idx", C.c_void_p)]

    @classmethod
    def run(cls, off=0):
        return cls(RUN, int(off), 0, None)

    @classmethod
    def gap(cls, split, off0, off1):
        return cls(int(split), int(off0), int(off1), None)


class GemmDesc(C.Structure):
    """``ibmi_gemm_desc`` (include/ibmi_b200.h)."""
    _fields_ = [
        ("x", C.c_void_p), ("ldx", C.c_int64), ("xm", Map), ("xrows", C.c_int64), ("xcols", C.c_int64),
        ("y", C.c_void_p), ("ldy", C.c_int64), ("yn", Map), ("yrows", C.c_int64), ("ycols", C.c_int64),
        ("m", C.c_int64), ("n", C.c_int64),
        ("nseg", C.c_int), ("seg_x0", C.c_int64 * 2), ("seg_y0", C.c_int64 * 2), ("seg_len", C.c_int64 * 2),
        ("c", C.c_void_p), ("ldc", C.c_int64), ("cm", Map), ("cn", Map), ("cidx", C.c_void_p), ("direct", C.c_int),
        ("c2", C.c_void_p), ("ldc2", C.c_int64), ("c2m", Map), ("c2n", Map), ("mirror", C.c_int),
        ("alpha", C.c_double), ("beta", C.c_double), ("d", C.c_void_p), ("ldd", C.c_int64), ("dm", Map),
        ("dn", Map),
        ("lower", C.c_int), ("tma_safe", C.c_int), ("splits", C.c_int),
        ("frob_out", C.c_void_p),
        ("ws", C.c_void_p), ("ws_len", C.c_int64),
        ("peers", C.c_void_p), ("bc_panel", C.c_int64), ("bc_world", C.c_int), ("bc_rank", C.c_int),
        ("xt", C.c_int), ("yt", C.c_int),
    ]
