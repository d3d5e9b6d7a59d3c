"""Device-resident IBMI state: one ``ibmi_ctx`` of the CUDA library.

:class:`DeviceSolver` owns A, Σ, the per-set caches (A_II⁻¹, W) and the
estimate buffers in HBM, and exposes the sweep pieces the reference's
``solve`` loop is made of (`/root/reference/pkg/src/ibmi/solver.py:241-270`).
Non-contiguous partitions whose sets are pairwise disjoint (red-black,
custom disjoint JSON) are relabelled so every set is a run (the sweep is
permutation-equivariant: Σ(PAPᵀ) = PΣ(A)Pᵀ); Σ is mapped back on the way out.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi
from .partition import Partition, block_permutation, complement, contiguous_ranges

RESTART_SEED = 0x5EED   # reference linalg.py:49


def restart_vector(n: int) -> np.ndarray:
    """The normalised ``default_rng(0x5EED)`` draw of linalg.py:240-241."""
    v = np.random.default_rng(RESTART_SEED).standard_normal(n)
    return np.ascontiguousarray(v / np.linalg.norm(v))


class _FileMatrix:
    """Marker: A comes from an IBMI1 file (read by the library, not by Python)."""

    def __init__(self, path, p):
        self.path, self.p = str(path), int(p)
        self.shape = (self.p, self.p)


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda", False))


def _torch_stream_done(t) -> None:
    """Wait for torch's current stream on ``t``'s device.

    The library works on its own stream; a device tensor handed to it (or a
    block torch just allocated for it to fill) may still be produced or read
    by kernels queued on torch's stream, so that stream is drained before the
    library's device-to-device copy reads or writes the tensor."""
    import torch

    torch.cuda.current_stream(t.device).synchronize()


class DeviceSolver:
    """IBMI state for one solve on one GPU.

    ``a`` is a float64 numpy array (copied host→device) or a float64 CUDA
    torch tensor (copied device→device).  ``ranges`` is a list of ``(lo, hi)``
    runs, or pass ``partition=`` to derive them (and a relabelling if needed).
    """

    @classmethod
    def from_ibmi1(cls, path: str, partition: Partition, *, device: int = 0, stream: int | None = None):
        """Load A from an IBMI1 file straight into HBM (no host copy).  Only
        partitions that need no relabelling (runs or index lists) qualify."""
        from .matio import read_header

        rows, cols = read_header(path)
        if rows != cols or rows != partition.p:
            from .exceptions import DimensionMismatch

            raise DimensionMismatch(f"matrix shape ({rows}, {cols}) does not match partition over {partition.p}")
        return cls(_FileMatrix(path, rows), partition=partition, device=device, stream=stream)

    def __init__(self, a, ranges=None, *, partition: Partition | None = None, device: int = 0,
                 stream: int | None = None, perm: np.ndarray | None = None):
        L = _abi.lib()
        self._L = L
        self.device = int(device)
        self.perm = None
        self.general = None        # list of ascending index arrays (overlapping non-contiguous sets)
        if partition is not None:
            ranges = contiguous_ranges(partition)
            if ranges is None:
                bp = block_permutation(partition)
                if bp is not None:
                    self.perm, ranges = bp          # disjoint sets: relabel into runs
                else:
                    self.general = [np.unique(np.asarray(s, dtype=np.int64)) for s in partition.sets]
                    ranges = [(int(s[0]), int(s[-1]) + 1) for s in self.general]
        elif perm is not None:
            self.perm = np.asarray(perm, dtype=np.int64)
        if ranges is None:
            raise ValueError("need ranges or partition")
        self.ranges = [(int(lo), int(hi)) for lo, hi in ranges]
        self.sizes = [len(s) for s in self.general] if self.general else [hi - lo for lo, hi in self.ranges]
        on_dev = _is_cuda_tensor(a)
        from_file = isinstance(a, _FileMatrix)
        if from_file:
            if self.perm is not None:
                raise NotImplementedError("relabelled partitions need A in memory; load it with matio.load_matrix")
            p, lda = a.p, a.p
        elif on_dev:
            import torch

            if a.dtype != torch.float64:
                a = a.to(torch.float64)
            if a.stride(1) != 1:
                a = a.contiguous()
            if self.perm is not None:
                idx = torch.as_tensor(self.perm, device=a.device)
                a = a.index_select(0, idx).index_select(1, idx).contiguous()
            p, lda = a.shape[0], a.stride(0)
            self._a_keep = a
        else:
            a = np.asarray(a, dtype=np.float64)
            if self.perm is not None:
                a = a[np.ix_(self.perm, self.perm)]
            a = np.ascontiguousarray(a)
            p, lda = a.shape[0], a.shape[1]
        self.p = int(p)
        h = C.c_void_p()
        _abi.check(L.ibmi_create(C.byref(h), self.device, self.p, C.c_void_p(stream or 0)), "ibmi_create")
        self._h = h
        try:
            if from_file:
                _abi.check(L.ibmi_load_ibmi1(h, a.path.encode()), "load_ibmi1")
            else:
                if on_dev:
                    _torch_stream_done(a)
                _abi.check(L.ibmi_set_matrix(h, C.c_void_p(_abi.dptr(a)), lda, int(on_dev)), "set_matrix")
            k = len(self.ranges)
            if self.general:
                ptr = np.zeros(k + 1, dtype=np.int64)
                ptr[1:] = np.cumsum([len(s) for s in self.general])
                idx = np.ascontiguousarray(np.concatenate(self.general))
                _abi.check(L.ibmi_set_partition_general(h, k, ptr.ctypes.data_as(C.POINTER(C.c_int64)),
                                                        idx.ctypes.data_as(C.POINTER(C.c_int64))), "set_partition")
            else:
                lo = (C.c_int64 * k)(*[r[0] for r in self.ranges])
                hi = (C.c_int64 * k)(*[r[1] for r in self.ranges])
                _abi.check(L.ibmi_set_partition(h, k, lo, hi), "set_partition")
            self._restart_n = None
            self._set_restart(self.p - self.sizes[-1])
        except BaseException:
            self.close()
            raise
        self._a_keep = None

    # -- lifecycle
    def close(self):
        if getattr(self, "_h", None):
            self._L.ibmi_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stream_handle(self) -> int:
        """The context's CUDA stream (``cudaStream_t`` as an int)."""
        st = C.c_void_p()
        _abi.check(self._L.ibmi_context_stream(self._h, C.byref(st)), "context_stream")
        return st.value or 0

    # -- pieces
    def _set_restart(self, n: int):
        if n >= 1 and n != self._restart_n:
            v = restart_vector(n)
            _abi.check(self._L.ibmi_set_restart_vector(self._h, n, _abi.dbl_ptr(v)), "set_restart_vector")
            self._restart_n = n

    def set_emulation(self, moduli: int):
        """0: FP64 DMMA GEMMs; 8..20: Ozaki-II emulation with that many moduli."""
        _abi.check(self._L.ibmi_set_emulation(self._h, int(moduli)), "set_emulation")

    @property
    def emulation(self) -> int:
        n = C.c_int()
        _abi.check(self._L.ibmi_get_emulation(self._h, C.byref(n)), "get_emulation")
        return n.value

    def setup(self, first: int = 0, count: int = -1):
        fs, fp = C.c_int(-1), C.c_int64(-1)
        rc = self._L.ibmi_setup(self._h, first, count, C.byref(fs), C.byref(fp))
        _abi.check(rc, "setup", fail_set=fs.value, fail_pivot=fp.value)

    def init_sigma(self, kind: int = _abi.GUESS_IDENTITY, guess: np.ndarray | None = None):
        """Σ = I, Σ[c₁,c₁] = guess block.  GUESS_MATRIX: ``guess`` is that block (ascending
        complement order); GUESS_MC: ``guess`` is the p × n matrix of standard-normal draws."""
        if kind == _abi.GUESS_MC:
            w = np.ascontiguousarray(np.asarray(guess, dtype=np.float64))
            if self.perm is not None:
                raise ValueError("GUESS_MC needs the original ordering; pass the block via GUESS_MATRIX")
            _abi.check(self._L.ibmi_init_sigma(self._h, kind, C.c_void_p(w.ctypes.data), w.shape[1], 0), "init_sigma")
            return
        if kind == _abi.GUESS_MATRIX:
            g = np.ascontiguousarray(np.asarray(guess, dtype=np.float64))
            if self.perm is not None:
                g = self._permute_guess(g)
            _abi.check(self._L.ibmi_init_sigma(self._h, kind, C.c_void_p(g.ctypes.data), g.shape[1], 0), "init_sigma")
        else:
            _abi.check(self._L.ibmi_init_sigma(self._h, kind, None, 0, 0), "init_sigma")

    def _permute_guess(self, g):  # noqa: D401
        # guess is over the ascending original complement of set 0; the
        # device complement of set 0 is perm[[0,lo) ∪ [hi,p)] in that order.
        lo, hi = self.ranges[0]
        dev_c = np.concatenate([self.perm[:lo], self.perm[hi:]])
        order = np.argsort(np.argsort(dev_c))   # rank of each device index in the ascending list
        return np.ascontiguousarray(g[np.ix_(order, order)])

    def set_sigma(self, s):
        if _is_cuda_tensor(s):
            import torch

            s = s.to(torch.float64).contiguous()
            if self.perm is not None:
                idx = torch.as_tensor(self.perm, device=s.device)
                s = s.index_select(0, idx).index_select(1, idx).contiguous()
            _torch_stream_done(s)
            _abi.check(self._L.ibmi_set_sigma(self._h, C.c_void_p(s.data_ptr()), s.stride(0), 1), "set_sigma")
            return
        s = np.asarray(s, dtype=np.float64)
        if self.perm is not None:
            s = s[np.ix_(self.perm, self.perm)]
        s = np.ascontiguousarray(s)
        _abi.check(self._L.ibmi_set_sigma(self._h, C.c_void_p(s.ctypes.data), s.shape[1], 0), "set_sigma")

    def sigma(self, out: np.ndarray | None = None, on_device: bool = False):
        """Σ as a host numpy array (default) or a CUDA torch tensor."""
        if on_device:
            import torch

            t = torch.empty((self.p, self.p), dtype=torch.float64, device=f"cuda:{self.device}")
            _torch_stream_done(t)
            _abi.check(self._L.ibmi_get_sigma(self._h, C.c_void_p(t.data_ptr()), self.p, 1), "get_sigma")
            if self.perm is not None:
                inv = torch.as_tensor(np.argsort(self.perm), device=t.device)
                t = t.index_select(0, inv).index_select(1, inv)
            return t
        host = np.empty((self.p, self.p)) if (out is None or self.perm is not None) else out
        _abi.check(self._L.ibmi_get_sigma(self._h, C.c_void_p(host.ctypes.data), host.shape[1], 0), "get_sigma")
        if self.perm is not None:
            inv = np.argsort(self.perm)
            host = host[np.ix_(inv, inv)]
            if out is not None:
                out[...] = host
                return out
        return host

    def sigma_view(self):
        """Zero-copy CUDA tensor over the context's Σ (p × p view of the p × ld buffer, in
        the context's own index order).  For sizes where a copy does not fit next to the
        solve (c5: 34 GB); valid until ``close`` and only after the context's stream is
        synchronised."""
        import torch

        if self.perm is not None:
            raise ValueError("sigma_view is in the relabelled order; use sigma() for permuted partitions")
        ptr, r, c, ld = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int64()
        _abi.check(self._L.ibmi_export(self._h, 1, 0, C.byref(ptr), C.byref(r), C.byref(c), C.byref(ld)), "export")
        torch.cuda.synchronize(self.device)

        class _View:
            __cuda_array_interface__ = {"shape": (int(r.value), int(c.value)), "typestr": "<f8",
                                        "data": (int(ptr.value), False), "strides": (int(ld.value) * 8, 8),
                                        "version": 3}

        return torch.as_tensor(_View(), device=f"cuda:{self.device}")

    def block_update(self, k: int):
        _abi.check(self._L.ibmi_block_update(self._h, int(k)), "block_update")

    def error_estimate(self, k: int, rtol: float, max_iters: int):
        self._set_restart(self.p - self.sizes[k])
        e, it, cv = C.c_double(), C.c_int(), C.c_int()
        _abi.check(self._L.ibmi_error_estimate(self._h, int(k), float(rtol), int(max_iters), C.byref(e),
                                               C.byref(it), C.byref(cv)), "error_estimate")
        return e.value, it.value, bool(cv.value)

    def sweep(self, rtol: float, max_iters: int):
        self._set_restart(self.p - self.sizes[-1])
        e, it, cv = C.c_double(), C.c_int(), C.c_int()
        _abi.check(self._L.ibmi_sweep(self._h, float(rtol), int(max_iters), C.byref(e), C.byref(it), C.byref(cv)),
                   "sweep")
        return e.value, it.value, bool(cv.value)

    def sweep_timed(self, rtol: float, max_iters: int):
        """Sweep without the graph, returning per-kernel-class device ms."""
        self._set_restart(self.p - self.sizes[-1])
        e, it, cv = C.c_double(), C.c_int(), C.c_int()
        t = (C.c_float * 6)()
        _abi.check(self._L.ibmi_sweep_timed(self._h, float(rtol), int(max_iters), C.byref(e), C.byref(it),
                                            C.byref(cv), t), "sweep_timed")
        keys = ("panel_gemm", "diag_gemm", "estimate_gemm", "gram_gemm", "power_iteration", "sweep")
        return e.value, it.value, bool(cv.value), dict(zip(keys, list(t)))

    def solve_loop(self, tol: float, max_sweeps: int, rtol: float, max_iters: int, stopping: str = "estimate",
                   residual_every_sweep: bool = False):
        """Whole solve loop on the device (``ibmi_solve_loop``): returns a dict of
        per-sweep traces, or raises NotImplementedError if the graph cannot be built."""
        self._set_restart(self.p - self.sizes[-1])
        n = int(max_sweeps)
        err = np.zeros(n)
        res = np.zeros(n)
        ms = np.zeros(n)
        pit = np.zeros(n, dtype=np.int32)
        pcv = np.zeros(n, dtype=np.int32)
        sw, cv = C.c_int(), C.c_int()
        ip = C.POINTER(C.c_int)
        mode = 0 if stopping != "frobenius" else (2 if residual_every_sweep else 1)
        _abi.check(self._L.ibmi_solve_loop(self._h, float(tol), n, float(rtol), int(max_iters),
                                           mode, C.byref(sw), C.byref(cv),
                                           _abi.dbl_ptr(err), pit.ctypes.data_as(ip), pcv.ctypes.data_as(ip),
                                           _abi.dbl_ptr(res), _abi.dbl_ptr(ms)), "solve_loop")
        k = sw.value
        return dict(sweeps=k, converged=bool(cv.value), error_trace=err[:k].tolist(), power_iters=pit[:k].tolist(),
                    power_conv=pcv[:k].astype(bool).tolist(),
                    residual_trace=res[:k].tolist() if stopping == "frobenius" else [],
                    sweep_seconds=(ms[:k] * 1e-3).tolist())

    def frobenius(self) -> float:
        out = C.c_double()
        _abi.check(self._L.ibmi_frobenius_residual(self._h, C.byref(out)), "frobenius_residual")
        return out.value

    def save_sigma_ibmi1(self, path: str):
        """Σ from HBM straight to an IBMI1 file (original index order)."""
        if self.perm is not None:
            from .matio import save_ibmi

            save_ibmi(path, self.sigma())
            return
        _abi.check(self._L.ibmi_save_sigma_ibmi1(self._h, str(path).encode()), "save_sigma_ibmi1")

    def device_bytes(self) -> int:
        b = C.c_int64()
        _abi.check(self._L.ibmi_device_bytes(self._h, C.byref(b)))
        return b.value


def probe_fp64_peak(device: int = 0) -> float:
    """Measured DMMA FP64 throughput in TFLOP/s (roofline denominator)."""
    out = C.c_double()
    _abi.check(_abi.lib().ibmi_probe_fp64_peak(int(device), C.byref(out)), "probe_fp64_peak")
    return out.value


def complement_of(part: Partition, j: int) -> np.ndarray:
    return complement(part, j)
