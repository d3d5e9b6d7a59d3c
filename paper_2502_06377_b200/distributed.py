"""Sharded IBMI sweep over several GPUs.

One process per GPU, ``torch.distributed`` for the plumbing (NCCL on GPUs).

Layout.  Σ is stored as block-cyclic **row panels** of ``panel`` rows: global
row r lives on rank ``(r // panel) % world``.  Because Σ is symmetric these are
also its column panels.  A, W_k = A_II⁻¹A_Ic and A_II⁻¹ are replicated.  The
set-up kernels run on every rank: they are a few percent of a solve, cheaper
than broadcasting W (42 GB at c5).

One block update of set I = [lo, hi) on rank g (the reference's
``_BlockOp.apply``, solver.py:122-129, split by columns):

1. panel GEMM ``Mbuf = −W·Σ[c ∩ own_g, c]ᵀ`` (b × |c ∩ own_g|).  Its mirrored
   epilogue writes ``Σ[c ∩ own_g, I] = −Mᵀ`` straight into the local panel;
2. partial ``top_g = −Mbuf·W[:, c ∩ own_g]ᵀ`` → ``all_reduce`` → every rank
   holds ``Σ_II = sym(A_II⁻¹ + M Wᵀ)`` and stores its own rows of it;
3. exchange: the owner of row i ∈ I needs ``Σ[i, c] = −M[i, :]``, whose
   columns are spread over all ranks → one ``all_to_all`` of b×c doubles.

Error estimate (solver.py:147-155): the owners of I's rows compute their rows
of ``B = Σ[I,:]·A[:,c]`` locally (A is replicated), ``all_gather`` assembles
B, and the Gram power iteration runs replicated, giving the same σ on every
rank.  ‖I − AΣ‖_F: local rows of ``ΣA`` with the fused (δ − x)² epilogue, then
``all_reduce``.

Compute goes through a backend.  :class:`CudaBackend` (this module) calls
``libibmi_b200.so``.  The CPU tests inject a torch emulation, which lives in
``tests/`` and never in the product.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .device import DeviceSolver, restart_vector
from .partition import Partition, block_permutation, contiguous_ranges

__all__ = ["RowPanels", "GemmSpec", "CudaBackend", "ShardedSolver", "solve_sharded"]


# --------------------------------------------------------------------------- layout
class RowPanels:
    """Block-cyclic ownership of the p rows: row r → rank (r // panel) % world."""

    def __init__(self, p: int, world: int, panel: int = 128):
        self.p, self.world, self.panel = int(p), int(world), int(panel)
        r = np.arange(self.p, dtype=np.int64)
        self.owner = (r // self.panel) % self.world
        self.rows = [np.nonzero(self.owner == h)[0].astype(np.int64) for h in range(self.world)]

    def local_range(self, h: int, lo: int, hi: int) -> tuple[int, int]:
        """Local index range [a0, a1) of rank h's rows inside [lo, hi)."""
        rows = self.rows[h]
        return int(np.searchsorted(rows, lo)), int(np.searchsorted(rows, hi))


# --------------------------------------------------------------------------- GEMM spec
@dataclass
class GemmSpec:
    """Backend-neutral description of one NT GEMM (mirrors ``ibmi_gemm_desc``).

    Maps are ``(split, off0, off1)`` triples, or ``int`` for a plain run
    starting at that offset.  Tensors are 2-D with unit column stride.
    """

    x: object
    xm: object
    y: object
    yn: object
    m: int
    n: int
    segs: list                       # [(x0, y0, len), ...] (≤ 2)
    c: object = None
    cm: object = 0
    cn: object = 0
    cidx: object = None              # int64 tensor: direct-store / δ row index of m
    direct: bool = True
    c2: object = None
    c2m: object = 0
    c2n: object = 0
    mirror: bool = False
    alpha: float = 1.0
    beta: float = 0.0
    d: object = None
    dm: object = 0
    dn: object = 0
    lower: bool = False
    tma_safe: bool = False
    frob: bool = False               # return Σ (δ − acc)² instead of storing
    xrows: int = 0
    xcols: int = 0
    yrows: int = 0
    ycols: int = 0
    xt: bool = False                 # X given transposed: X(m, k) = x[seg.x0 + k][xm.off0 + m]
    yt: bool = False                 # Y given transposed: Y(n, k) = y[seg.y0 + k][yn.off0 + n]
    peers: object = None             # int64 tensor of per-rank Σ panel pointers (fused exchange)
    bc_panel: int = 0
    bc_world: int = 1
    bc_rank: int = 0
    extra: dict = field(default_factory=dict)


def _map3(m):
    if isinstance(m, (int, np.integer)):
        return (_abi.RUN, int(m), 0)
    return tuple(int(v) for v in m)


def _cmap(m):
    return _abi.Map(*_map3(m), None)


def map_indices(m, n: int) -> np.ndarray:
    """Materialise a map over logical indices 0..n-1 (used by emulation backends)."""
    split, off0, off1 = _map3(m)
    i = np.arange(n, dtype=np.int64)
    return np.where(i < split, off0 + i, off1 + (i - split))


# --------------------------------------------------------------------------- CUDA backend
class _CudaArray:
    def __init__(self, ptr, rows, cols, ld):
        self.__cuda_array_interface__ = {"shape": (int(rows), int(cols)), "typestr": "<f8",
                                         "data": (int(ptr), False), "strides": (int(ld) * 8, 8), "version": 3}


class CudaBackend:
    """Compute through libibmi_b200.so on the current CUDA device."""

    def __init__(self, device: int):
        import torch

        self.torch = torch
        self.device = torch.device(f"cuda:{device}")
        self.L = _abi.lib()
        self._ctx = None
        self._ws = None

    # set-up: the single-GPU context does the per-set Cholesky / inverse / W
    def setup(self, a, ranges):
        torch = self.torch
        self._ctx = DeviceSolver(a, ranges, device=self.device.index,
                                 stream=torch.cuda.current_stream(self.device).cuda_stream)
        self._ctx.setup()
        h = self._ctx._h

        def view(which, k=0):
            ptr, r, c, ld = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int64()
            _abi.check(self.L.ibmi_export(h, which, k, C.byref(ptr), C.byref(r), C.byref(c), C.byref(ld)), "export")
            return torch.as_tensor(_CudaArray(ptr.value, r.value, c.value, ld.value), device=self.device)

        A = view(0)
        W = [view(2, k) for k in range(len(ranges))]
        ainv = [view(3, k) for k in range(len(ranges))]
        return A, W, ainv

    def zeros(self, *shape):
        return self.torch.zeros(shape, dtype=self.torch.float64, device=self.device)

    def index_tensor(self, idx):
        return self.torch.as_tensor(np.asarray(idx, dtype=np.int64), device=self.device)

    # operand-sharded set-up (ShardedSolver, operands="sharded"): primitives only
    def upload_rows(self, a, rows):
        """Device copy of ``a[rows, :]`` with the leading dimension padded to 32 doubles
        (16-byte aligned rows for TMA; padding columns are zero)."""
        torch = self.torch
        n, p = len(rows), int(a.shape[1])
        out = torch.zeros((max(n, 1), -(-p // 32) * 32), dtype=torch.float64, device=self.device)
        if n:
            if hasattr(a, "is_cuda"):
                out[:n, :p] = a.to(self.device, torch.float64).index_select(0, self.index_tensor(rows))
            else:
                out[:n, :p] = torch.from_numpy(np.ascontiguousarray(np.asarray(a, dtype=np.float64)[rows, :]))
        return out[:n, :p] if n else out[:0, :p]

    def transposed(self, t):
        """Contiguous transpose of a 2-D device tensor, rows padded to 32 doubles (TMA alignment)."""
        r, c = t.shape
        out = self.torch.zeros((max(c, 1), -(-max(r, 1) // 32) * 32), dtype=self.torch.float64, device=self.device)
        out[:c, :r] = t.t()
        return out[:c, :r]

    def spd_inverse(self, blk):
        """A_II⁻¹ on the device (linalg.py:122-130): symmetric check (linalg.py:68-77),
        blocked Cholesky + inverse; raises NotPositiveDefinite(index) like the reference."""
        from . import linalg

        torch = self.torch
        if not hasattr(blk, "is_cuda"):
            blk = torch.from_numpy(np.ascontiguousarray(np.asarray(blk, dtype=np.float64)))
        d = blk.to(self.device, torch.float64).contiguous()
        scale = float(d.abs().max()) if d.numel() else 0.0
        if scale != 0.0 and float((d - d.t()).abs().max()) > linalg.SYMMETRY_RTOL * scale:
            raise ValueError("matrix is not symmetric")
        return linalg.spd_inverse(d, self.device.index)

    def sym_rows(self, base, low, rel, dst):
        """dst[i, :] = base[rel[i], :] + symmetric completion of the lower triangle ``low``."""
        n = base.shape[0]
        stream = C.c_void_p(self.torch.cuda.current_stream(self.device).cuda_stream)
        _abi.check(self.L.ibmi_sym_rows(C.c_void_p(base.data_ptr()), base.stride(0), C.c_void_p(low.data_ptr()),
                                        low.stride(0), C.c_void_p(rel.data_ptr()), rel.numel(), n,
                                        C.c_void_p(dst.data_ptr()), dst.stride(0), stream), "sym_rows")

    def gemm(self, s: GemmSpec):
        torch = self.torch
        d = _abi.GemmDesc()
        d.x, d.ldx, d.xm = s.x.data_ptr(), s.x.stride(0), _cmap(s.xm)
        d.xrows, d.xcols = s.xrows or s.x.shape[0], s.xcols or s.x.shape[1]
        d.y, d.ldy, d.yn = s.y.data_ptr(), s.y.stride(0), _cmap(s.yn)
        d.yrows, d.ycols = s.yrows or s.y.shape[0], s.ycols or s.y.shape[1]
        d.m, d.n = int(s.m), int(s.n)
        segs = [g for g in s.segs if g[2] > 0]
        d.nseg = len(segs)
        for i, (x0, y0, ln) in enumerate(segs):
            d.seg_x0[i], d.seg_y0[i], d.seg_len[i] = int(x0), int(y0), int(ln)
        if s.c is not None:
            d.c, d.ldc = s.c.data_ptr(), s.c.stride(0)
        d.cm, d.cn = _cmap(s.cm), _cmap(s.cn)
        d.cidx = s.cidx.data_ptr() if s.cidx is not None else None
        d.direct = int(bool(s.direct) and not s.frob)
        if s.mirror:
            d.mirror = 1
            if s.c2 is not None:
                d.c2, d.ldc2 = s.c2.data_ptr(), s.c2.stride(0)
                d.c2m, d.c2n = _cmap(s.c2m), _cmap(s.c2n)
        d.alpha, d.beta = float(s.alpha), float(s.beta)
        if s.d is not None:
            d.d, d.ldd = s.d.data_ptr(), s.d.stride(0)
            d.dm, d.dn = _cmap(s.dm), _cmap(s.dn)
        d.lower, d.tma_safe, d.splits = int(s.lower), int(s.tma_safe), 0     # 0: automatic split-K
        d.xt, d.yt = int(s.xt), int(s.yt)
        if s.peers is not None:
            d.peers, d.bc_panel, d.bc_world, d.bc_rank = s.peers.data_ptr(), s.bc_panel, s.bc_world, s.bc_rank
        out = None
        if s.frob:
            out = torch.zeros(2, dtype=torch.float64, device=self.device)
            d.frob_out = out.data_ptr()
        need = C.c_int64()
        _abi.check(self.L.ibmi_gemm_workspace(C.byref(d), C.byref(need)), "gemm_workspace")
        if need.value:
            if self._ws is None or self._ws.numel() < need.value:
                self._ws = torch.empty(need.value, dtype=torch.float64, device=self.device)
            d.ws, d.ws_len = self._ws.data_ptr(), self._ws.numel()
        stream = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _abi.check(self.L.ibmi_gemm(C.byref(d), stream), "gemm")
        return out[1] if s.frob else None

    def gemm_xt(self, x, x_col0, y, m, n, segs, c, alpha=1.0):
        """C = alpha · X · Yᵀ with X(m, k) = x[x0 + k][x_col0 + m] (x read transposed)."""
        self.gemm(GemmSpec(x=x, xm=x_col0, y=y, yn=0, m=m, n=n, segs=segs, c=c, alpha=alpha, xt=True,
                           xrows=x.shape[0], xcols=x.shape[1], yrows=y.shape[0], ycols=y.shape[1]))

    # peer-visible Σ panels for the fused exchange
    def alloc_shared(self, rows, cols):
        ptr = C.c_void_p()
        _abi.check(self.L.ibmi_device_alloc(self.device.index, int(rows) * int(cols) * 8, C.byref(ptr)), "device_alloc")
        self._shared = getattr(self, "_shared", []) + [ptr.value]
        t = self.torch.as_tensor(_CudaArray(ptr.value, rows, cols, cols), device=self.device)
        h = C.create_string_buffer(64)
        _abi.check(self.L.ibmi_ipc_handle(C.c_void_p(ptr.value), h), "ipc_handle")
        return t, bytes(h.raw)

    def open_peer(self, handle: bytes) -> int:
        ptr = C.c_void_p()
        _abi.check(self.L.ibmi_ipc_open(self.device.index, handle, C.byref(ptr)), "ipc_open")
        self._opened = getattr(self, "_opened", []) + [ptr.value]
        return ptr.value

    def rows_to_host(self, t, out: np.ndarray, host_rows: np.ndarray):
        """out[host_rows[r], :] = t[r, :] through the library's pinned staging pool."""
        torch = self.torch
        rows = np.ascontiguousarray(host_rows, dtype=np.int64)
        assert out.dtype == np.float64 and out.flags.c_contiguous and t.stride(1) == 1
        stream = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _abi.check(self.L.ibmi_copy_rows(self.device.index, C.c_void_p(t.data_ptr()), t.stride(0),
                                         out.ctypes.data_as(C.c_void_p), out.shape[1], t.shape[0], t.shape[1],
                                         rows.ctypes.data_as(C.c_void_p), 0, stream), "copy_rows")

    def two_norm(self, b, rtol, max_iters):
        torch = self.torch
        v = restart_vector(b.shape[1])
        sig, it, cv = C.c_double(), C.c_int(), C.c_int()
        stream = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _abi.check(self.L.ibmi_two_norm(b.shape[0], b.shape[1], C.c_void_p(b.data_ptr()), b.stride(0),
                                        _abi.dbl_ptr(v), float(rtol), int(max_iters), C.byref(sig), C.byref(it),
                                        C.byref(cv), stream), "two_norm")
        return sig.value, it.value, bool(cv.value)

    def two_norm_gram(self, b, g, y1, rtol, max_iters):
        """‖b‖₂ from the caller's Gram matrix g = b·bᵀ and y₁ = b·(1/√cols) (rows ≤ cols)."""
        torch = self.torch
        v = restart_vector(b.shape[1])
        sig, it, cv = C.c_double(), C.c_int(), C.c_int()
        stream = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _abi.check(self.L.ibmi_two_norm_gram(b.shape[0], b.shape[1], C.c_void_p(b.data_ptr()), b.stride(0),
                                             C.c_void_p(g.data_ptr()), g.stride(0), C.c_void_p(y1.data_ptr()),
                                             _abi.dbl_ptr(v), float(rtol), int(max_iters), C.byref(sig),
                                             C.byref(it), C.byref(cv), stream), "two_norm_gram")
        return sig.value, it.value, bool(cv.value)

    def close(self):
        self.torch.cuda.synchronize(self.device)
        for ptr in getattr(self, "_opened", []):
            self.L.ibmi_ipc_close(C.c_void_p(ptr))
        self._opened = []
        for ptr in getattr(self, "_shared", []):
            self.L.ibmi_device_free(C.c_void_p(ptr))
        self._shared = []
        if self._ctx is not None:
            self._ctx.close()
            self._ctx = None


# --------------------------------------------------------------------------- collectives
class _Done:
    def wait(self):
        return True


class _Comm:
    """torch.distributed calls, staging CUDA tensors through the host when the
    process group cannot take them (gloo)."""

    def __init__(self, group):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.backend = dist.get_backend(group)
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def _stage(self, t):
        return self.backend == "gloo" and t.is_cuda

    def all_reduce(self, t):
        if self.world == 1:
            return t
        if self._stage(t):
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            self.dist.all_reduce(t, group=self.group)
        return t

    def barrier(self):
        """Stream-ordered barrier (a one-element all-reduce)."""
        if self.world == 1:
            return
        if getattr(self, "_tok", None) is None:
            self._tok = self.torch.zeros(1, dtype=self.torch.float64,
                                         device="cpu" if self.backend == "gloo" else "cuda")
        self.all_reduce(self._tok)

    def all_to_all(self, out, inp, out_splits, in_splits):
        if self.world == 1:
            out.copy_(inp)
            return out
        if self._stage(inp):
            ho = out.cpu()
            self.dist.all_to_all_single(ho, inp.cpu(), out_splits, in_splits, group=self.group)
            out.copy_(ho)
        else:
            self.dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
        return out

    def broadcast(self, t, src: int):
        """In-place broadcast of ``t`` from group rank ``src``."""
        if self.world == 1:
            return t
        gsrc = self.dist.get_global_rank(self.group, src) if self.group is not None else src
        if self._stage(t):
            h = t.cpu()
            self.dist.broadcast(h, src=gsrc, group=self.group)
            if self.rank != src:
                t.copy_(h)
        else:
            self.dist.broadcast(t, src=gsrc, group=self.group)
        return t

    def all_gather_start(self, out, inp):
        """Start ``out[h] = inp of rank h`` (equal shapes; out is (world, *inp.shape)).
        Returns a handle whose ``wait()`` orders the result before the caller's
        later work.  NCCL: asynchronous on the communicator's stream, so the gather
        overlaps kernels launched afterwards; gloo: done on return."""
        if self.world == 1:
            out[0].copy_(inp)
            return _Done()
        if self._stage(inp):
            ho = out.cpu()
            self.dist.all_gather_into_tensor(ho.view(-1), inp.cpu().contiguous().view(-1), group=self.group)
            out.copy_(ho)
            return _Done()
        return self.dist.all_gather_into_tensor(out.view(-1), inp.contiguous().view(-1), group=self.group,
                                                async_op=True)

    def all_gather_rows(self, t, counts):
        """Concatenate every rank's rows (rank order); counts[h] = rows of rank h."""
        torch = self.torch
        if self.world == 1:
            return t
        mx = max(counts)
        pad = torch.zeros((mx, t.shape[1]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        stage = self._stage(pad)
        src = pad.cpu() if stage else pad
        outs = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(outs, src, group=self.group)
        out = torch.cat([o[:c] for o, c in zip(outs, counts)], dim=0)
        return out.to(t.device) if stage else out


# --------------------------------------------------------------------------- solver
class ShardedSolver:
    """IBMI state sharded by block-cyclic row panels over a process group.

    Every rank passes the same ``a`` (host array or its own device copy) and
    partition.  Set ranges must be contiguous runs; pairwise-disjoint
    non-contiguous sets are relabelled first, as on one GPU.
    """

    def __init__(self, a, partition: Partition | None = None, ranges=None, *, group=None, panel: int = 128,
                 backend=None, device: int | None = None, exchange: str = "auto", operands: str = "auto"):
        import torch
        import torch.distributed as dist

        self.torch = torch
        group = group or dist.group.WORLD
        self.comm = _Comm(group)
        self.rank, self.world = self.comm.rank, self.comm.world
        self.perm = None
        if partition is not None:
            ranges = contiguous_ranges(partition)
            if ranges is None:
                bp = block_permutation(partition)
                if bp is None:
                    raise NotImplementedError("overlapping non-contiguous partitions are not supported")
                self.perm, ranges = bp
                a = np.asarray(a, dtype=np.float64)[np.ix_(self.perm, self.perm)]
        self.ranges = [(int(lo), int(hi)) for lo, hi in ranges]
        self.p = int(a.shape[0])
        if backend is None:
            backend = CudaBackend(device if device is not None else torch.cuda.current_device())
        self.be = backend
        self.layout = RowPanels(self.p, self.world, panel)
        lay, g = self.layout, self.rank
        self.own = lay.rows[g]
        self.n_loc = len(self.own)
        self.n_max = max(len(r) for r in lay.rows)
        if operands == "auto":
            operands = "sharded" if self.world > 1 else "replicated"
        if operands not in ("replicated", "sharded"):
            raise ValueError(f"unknown operands mode {operands!r}")
        self.operands = operands
        self.own_t = backend.index_tensor(self.own)
        self.rows_t = [backend.index_tensor(r) for r in lay.rows]
        if operands == "replicated":
            self.A, self.W, self.ainv = backend.setup(a, self.ranges)
            self.ld = self.A.stride(0)
        else:
            self._setup_sharded(a)
        if exchange == "auto":
            # fused peer-memory exchange when every rank is on this node (NVLink/NVSwitch)
            import socket

            names = [None] * self.world
            self.torch.distributed.all_gather_object(names, socket.gethostname(), group=self.comm.group)
            exchange = "p2p" if isinstance(backend, CudaBackend) and len(set(names)) == 1 else "nccl"
        if exchange not in ("nccl", "p2p"):
            raise ValueError(f"unknown exchange {exchange!r}")
        self.exchange = exchange
        if exchange == "p2p":
            # Σ panels live in IPC-exportable memory; every rank maps every peer's panel.
            # The mapping is agreed collectively: if any rank cannot map a peer, all ranks
            # fall back to the all_to_all exchange together (nobody is left in a collective).
            self.S, handle = backend.alloc_shared(max(self.n_loc, 1), self.ld)
            handles = [None] * self.world
            self.torch.distributed.all_gather_object(handles, handle, group=self.comm.group)
            ok = 1.0
            try:
                ptrs = [self.S.data_ptr() if h == self.rank else backend.open_peer(handles[h])
                        for h in range(self.world)]
            except Exception:          # noqa: BLE001 - any mapping failure -> collective fallback
                ok, ptrs = 0.0, None
            flag = self.torch.tensor([ok], dtype=self.torch.float64,
                                     device="cpu" if self.comm.backend == "gloo" else self.S.device)
            self.torch.distributed.all_reduce(flag, op=self.torch.distributed.ReduceOp.MIN, group=self.comm.group)
            if float(flag.item()) == 1.0:
                self.peers = backend.index_tensor(np.asarray(ptrs, dtype=np.uint64).view(np.int64))
            else:
                exchange = "nccl"
                self.S.zero_()
        else:
            self.S = backend.zeros(max(self.n_loc, 1), self.ld)
        self.exchange = exchange
        self.plan = [self._plan_set(lo, hi) for (lo, hi) in self.ranges]

    # ------------------------------------------------------------ operand-sharded set-up
    def _setup_sharded(self, a):
        """A, W_k and the set-up work split over the ranks (SURVEY §8(e) option B).

        Rank g keeps the row panel ``A[own_g, :]`` (= the column panel, A is
        symmetric) and the column shard ``W_k[:, own_g]`` of every set.  The K
        Cholesky / inverse jobs (solver.py:116-119) go round-robin over the ranks and
        each A_II⁻¹ (b × b) is broadcast; the W GEMM (solver.py:120) is local:
        ``W_k[:, own_g ∩ c] = A_II⁻¹ · A[I, own_g ∩ c]`` with ``A[I, j] = A[j, I]``
        read from the row panel.  Nothing of order p² is replicated."""
        from .exceptions import NotPositiveDefinite

        torch, be, lay, g = self.torch, self.be, self.layout, self.rank
        p = self.p
        if tuple(a.shape) != (p, p):
            from .exceptions import DimensionMismatch

            raise DimensionMismatch(f"expected a square matrix, got shape {tuple(a.shape)}")
        self.A = be.upload_rows(a, self.own)                      # n_loc × p view, padded ld
        self.AT = be.transposed(self.A)                           # p × n_loc: the column panel A[:, own_g], K-contiguous
        self.ld = -(-p // 32) * 32
        # (1) this rank's inverses; every rank learns every outcome before anyone raises
        mine, status = {}, []
        for k, (lo, hi) in enumerate(self.ranges):
            if k % self.world != g:
                continue
            try:
                mine[k] = be.spd_inverse(a[lo:hi, lo:hi])
            except NotPositiveDefinite as e:
                status.append((k, "spd", int(e.index)))
            except ValueError as e:
                status.append((k, "sym", str(e)))
        allst = [None] * self.world
        if self.world > 1:
            torch.distributed.all_gather_object(allst, status, group=self.comm.group)
        else:
            allst = [status]
        bad = sorted(x for st in allst for x in st)
        if bad:
            k, kind, info = bad[0]
            if kind == "spd":
                raise NotPositiveDefinite(info, set_index=k)
            raise ValueError(info)
        # (2) broadcast A_II⁻¹, form the local W shard
        self.ainv, self.Wg, self.W = [], [], None
        ldw = -(-max(self.n_max, 1) // 32) * 32
        for k, (lo, hi) in enumerate(self.ranges):
            b = hi - lo
            inv = mine.pop(k) if k in mine else be.zeros(b, b)
            self.comm.broadcast(inv, k % self.world)
            self.ainv.append(inv)
            a0, a1 = lay.local_range(g, lo, hi)
            wg = be.zeros(b, ldw)
            n_cl = self.n_loc - (a1 - a0)
            if n_cl > 0:
                # W[:, j] = Σ_i A_II⁻¹[:, i] · A[own_j, lo + i] for the local complement columns j
                be.gemm(GemmSpec(x=inv, xm=0, y=self.A, yn=(a0, 0, a1), m=b, n=n_cl, segs=[(0, lo, b)],
                                 c=wg, cm=0, cn=(a0, 0, a1), tma_safe=True, xrows=b, xcols=b,
                                 yrows=self.n_loc, ycols=p))
            self.Wg.append(wg)
        self._wfull = None
        self._wstage = None
        self._wpending = {}

    def _w_gather_start(self, k):
        """Begin the all-gather of W_k's column shards (the active block's panel
        broadcast).  W is static, so step k + 1's gather is started before step k's
        GEMMs and overlaps them on the communicator's stream."""
        if self.world == 1 or k in self._wpending:
            return
        bmax = max(hi - lo for lo, hi in self.ranges)
        ldw = self.Wg[k].shape[1]
        if self._wstage is None:
            self._wstage = [self.be.zeros(self.world, bmax, ldw) for _ in range(2)]
            self._wfull = self.be.zeros(bmax, self.ld)
        b = self.Wg[k].shape[0]
        st = self._wstage[k % 2]
        out = st.view(-1)[: self.world * b * ldw].view(self.world, b, ldw)
        self._wpending[k] = (self.comm.all_gather_start(out, self.Wg[k]), out)

    def _w_full(self, k):
        """W_k over all p columns in natural order (b × p view, zeros on I_k)."""
        if self.operands == "replicated":
            return self.W[k]
        if self.world == 1:
            return self.Wg[k]
        self._w_gather_start(k)
        work, out = self._wpending.pop(k)
        work.wait()
        b = self.Wg[k].shape[0]
        full = self._wfull[:b]
        for h in range(self.world):
            n_h = len(self.layout.rows[h])
            if n_h:
                full.index_copy_(1, self.rows_t[h], out[h][:, :n_h])
        return full

    # ------------------------------------------------------------ per-set plan
    def _plan_set(self, lo, hi):
        lay, g, be = self.layout, self.rank, self.be
        b, p = hi - lo, self.p
        a0, a1 = lay.local_range(g, lo, hi)
        n_cl = self.n_loc - (a1 - a0)
        ranges_all = [lay.local_range(h, lo, hi) for h in range(self.world)]
        rows_I = [lay.rows[h][r0:r1] for h, (r0, r1) in enumerate(ranges_all)]     # global rows of I per rank
        n_I = [len(r) for r in rows_I]
        send_perm = np.concatenate(rows_I) - lo if b else np.zeros(0, np.int64)   # M rows in destination order
        n_cl_all = [len(lay.rows[h]) - n_I[h] for h in range(self.world)]
        cols_c = []
        for h in range(self.world):
            r0, r1 = ranges_all[h]
            rr = lay.rows[h]
            cols_c.append(be.index_tensor(np.concatenate([rr[:r0], rr[r1:]])))
        return dict(lo=lo, hi=hi, b=b, a0=a0, a1=a1, n_cl=n_cl, n_I=n_I, n_cl_all=n_cl_all,
                    send_perm=be.index_tensor(send_perm),
                    my_rows_rel=be.index_tensor(rows_I[g] - lo), cols_c=cols_c, rows_I=rows_I)

    def _w_loc(self, k):
        """W_k restricted to this rank's columns, compact (zeros stay on I)."""
        if self.operands == "sharded":
            return self.Wg[k]
        cache = self.__dict__.setdefault("_wloc", {})
        if k not in cache:
            # one rank owns every column: W itself (its padding columns are never read)
            cache[k] = self.W[k] if self.n_loc == self.p else self.W[k].index_select(1, self.own_t).contiguous()
        return cache[k]

    # ------------------------------------------------------------ Σ₀
    def init_sigma(self, guess: str = "identity", sigma0_cc=None):
        """Σ = I, Σ[c₁,c₁] = identity or diag(1/A_ii) (solver.py:244-251 + BASELINE jacobi),
        or the given c₁ × c₁ matrix ``sigma0_cc`` (any other reference guess, solver.py:215-222,
        computed by the caller and identical on every rank)."""
        torch = self.torch
        self.S.zero_()
        if sigma0_cc is not None:
            lo, hi = self.ranges[0]
            comp = np.concatenate([np.arange(0, lo), np.arange(hi, self.p)])
            g = np.asarray(sigma0_cc, dtype=np.float64)
            if g.shape != (comp.size, comp.size):
                from .exceptions import DimensionMismatch

                raise DimensionMismatch(f"guess must be {comp.size} x {comp.size}, got {g.shape}")
            if self.perm is not None:
                raise NotImplementedError("explicit guesses with relabelled (non-contiguous) partitions")
            if self.n_loc:
                self._seed_sigma("identity")                      # the rows of I₁ keep their unit diagonal
                inc = (self.own < lo) | (self.own >= hi)          # my rows inside c₁
                pos = np.searchsorted(comp, self.own[inc])
                rows = self.be.index_tensor(np.nonzero(inc)[0])
                vals = torch.as_tensor(g[pos, :], device=self.S.device)
                blk = torch.zeros((len(pos), self.p), dtype=torch.float64, device=self.S.device)
                blk[:, self.be.index_tensor(comp)] = vals
                self.S[rows, : self.p] = blk
        elif self.n_loc:
            self._seed_sigma(guess)
        elif guess not in ("identity", "jacobi"):
            raise NotImplementedError(f"guess {guess!r} on the sharded path needs sigma0_cc")
        # No rank may start its first panel GEMM before every panel is seeded: in the
        # p2p exchange K1's epilogue stores −M into the OWNERS' panels, and a late
        # zero_() on a slow rank would wipe those stores.
        if self.world > 1:
            self.comm.barrier()

    def _seed_sigma(self, guess):
        torch = self.torch
        loc = torch.arange(self.n_loc, device=self.S.device)
        vals = torch.ones(self.n_loc, dtype=torch.float64, device=self.S.device)
        if guess == "jacobi":
            lo, hi = self.ranges[0]
            diag = self.A[self.own_t if self.operands == "replicated" else loc, self.own_t]
            inc = (self.own_t < lo) | (self.own_t >= hi)
            vals = torch.where(inc, 1.0 / diag, vals)
        elif guess != "identity":
            raise NotImplementedError(f"guess {guess!r} on the sharded path")
        self.S[loc, self.own_t] = vals

    # ------------------------------------------------------------ one block update
    def block_update(self, k: int):
        """One block step (solver.py:122-129) on the row panels.

        K1 (panel GEMM) writes Mbuf = −M (local columns), mirrors −Mᵀ into the
        local panel and — in the fused ``p2p`` mode — also stores −M straight
        into the owners' panels over NVLink.  K2 sums lower-triangle partials
        of M·Wᵀ (their sum is the lower triangle of the symmetric total)."""
        be, pl = self.be, self.plan[k]
        lo, hi, b, a0, a1, n_cl = pl["lo"], pl["hi"], pl["b"], pl["a0"], pl["a1"], pl["n_cl"]
        p = self.p
        p2p = self.exchange == "p2p"
        Mbuf = self._mbuf(b, n_cl)
        wfull = self._w_full(k)
        if self.operands == "sharded" and len(self.ranges) > 1:
            self._w_gather_start((k + 1) % len(self.ranges))     # prefetch: overlaps this step's GEMMs
        if n_cl > 0:
            spec = GemmSpec(x=wfull, xm=0, y=self.S, yn=(a0, 0, a1), m=b, n=n_cl,
                            segs=[(0, 0, lo), (hi, hi, p - hi)], c=Mbuf, cm=0, cn=0, mirror=True, c2=self.S,
                            c2m=lo, c2n=(a0, 0, a1), alpha=-1.0, tma_safe=True, xrows=b, xcols=p,
                            yrows=self.n_loc, ycols=p)
            if p2p:
                spec.peers, spec.bc_panel, spec.bc_world, spec.bc_rank = (self.peers, self.layout.panel,
                                                                          self.world, self.rank)
            be.gemm(spec)
        top = self._top(b)
        top.zero_()
        if n_cl > 0:
            be.gemm(GemmSpec(x=Mbuf, xm=0, y=self._w_loc(k), yn=0, m=b, n=b,
                             segs=[(0, 0, a0), (a0, a1, self.n_loc - a1)], c=top, alpha=-1.0, lower=True,
                             tma_safe=True, xrows=b, xcols=n_cl, yrows=b, ycols=self.n_loc))
        self.comm.all_reduce(top)     # in p2p mode also the barrier after which the peer stores have landed
        if a1 > a0:
            # Σ_II rows = ainv + the lower sum completed symmetrically, one kernel
            be.sym_rows(self.ainv[k], top, pl["my_rows_rel"], self.S[a0:a1, lo:hi])
        if p2p:
            # with overlapping sets the next step's peer stores hit rows of I_k ∩ I_{k+1}
            # that the Σ_II write above also touches: every rank must finish it first
            self.comm.barrier()
            return
        if self.world > 1:
            send = Mbuf[:, :n_cl].index_select(0, pl["send_perm"]).contiguous().reshape(-1)
            in_splits = [pl["n_I"][h] * n_cl for h in range(self.world)]
            my_I = pl["n_I"][self.rank]
            out_splits = [my_I * pl["n_cl_all"][h] for h in range(self.world)]
            recv = be.zeros(sum(out_splits))
            self.comm.all_to_all(recv, send, out_splits, in_splits)
            off = 0
            rows = self.S[a0:a1]
            for h in range(self.world):
                n = out_splits[h]
                if n:
                    blk = recv[off:off + n].view(my_I, pl["n_cl_all"][h])
                    rows.index_copy_(1, pl["cols_c"][h], blk)
                off += n
        elif a1 > a0 and n_cl > 0:
            self.S[a0:a1].index_copy_(1, pl["cols_c"][0], Mbuf[:, :n_cl])

    def _mbuf(self, b, n_cl):
        buf = getattr(self, "_mb", None)
        need = b * max(n_cl, 1)
        if buf is None or buf.numel() < need:
            self._mb = buf = self.be.zeros(need)
        return buf[:need].view(b, max(n_cl, 1))

    def _bbuf(self, b, c):
        buf = getattr(self, "_bb", None)
        if buf is None or buf.numel() < b * c:
            self._bb = buf = self.be.zeros(b * c)
        return buf[: b * c].view(b, c)

    def _top(self, b):
        buf = getattr(self, "_tb", None)
        if buf is None or buf.numel() < b * b:
            self._tb = buf = self.be.zeros(b * b)
        return buf[: b * b].view(b, b)

    # ------------------------------------------------------------ estimate
    def error_estimate(self, k: int, rtol: float = 1e-9, max_iters: int = 5000):
        """‖Σ_II A_Ic + Σ_Ic A_cc‖₂ (solver.py:147-155), same value on every rank."""
        torch, be, pl = self.torch, self.be, self.plan[k]
        lo, hi, b, a0, a1 = pl["lo"], pl["hi"], pl["b"], pl["a0"], pl["a1"]
        p, c = self.p, self.p - b
        if self.operands == "sharded":
            # B = Σ[I, :]·A[:, c] = Σ_g Σ[own_g, I]ᵀ · A[own_g, c]: both factors are columns of
            # the local row panels (a contraction over the local rows), then one all-reduce
            B = self._bbuf(b, c)
            B.zero_()
            if self.n_loc:
                # both operands K-contiguous (K = local rows): Σ[own_g, I]ᵀ is transposed per call
                # (b × n_loc, small), A[own_g, c]ᵀ = rows c of the static column panel AT
                sit = be.transposed(self.S[: self.n_loc, lo:hi])
                be.gemm(GemmSpec(x=sit, xm=0, y=self.AT, yn=(lo, 0, hi), m=b, n=c, segs=[(0, 0, self.n_loc)],
                                 c=B, cm=0, cn=0, tma_safe=True, xrows=b, xcols=self.n_loc, yrows=p,
                                 ycols=self.n_loc))
            self.comm.all_reduce(B)
            return self._two_norm_sharded(B, rtol, max_iters)
        Bloc = be.zeros(max(a1 - a0, 1), c)[: a1 - a0]
        if a1 > a0:
            be.gemm(GemmSpec(x=self.S, xm=a0, y=self.A, yn=(lo, 0, hi), m=a1 - a0, n=c, segs=[(0, 0, p)],
                             c=Bloc, tma_safe=True, xrows=self.n_loc, xcols=p, yrows=p, ycols=p))
        parts = self.comm.all_gather_rows(Bloc, pl["n_I"])
        order = np.argsort(np.concatenate(pl["rows_I"]), kind="stable")
        B = parts.index_select(0, be.index_tensor(order)).contiguous()
        return self._two_norm_sharded(B, rtol, max_iters)

    def _two_norm_sharded(self, B, rtol, max_iters):
        """‖B‖₂ with B (b × c) on every rank.  One rank: the library forms the Gram matrix.
        Several ranks (row form, b ≤ c): rank g forms ``B[:, chunk_g]·B[:, chunk_g]ᵀ`` over its
        share of the columns (lower tiles mirrored), one all-reduce of b × b sums them, and
        the power iteration runs replicated on the result — the b²·c Gram product is split G
        ways instead of repeated on every rank.  Same σ on every rank (identical inputs)."""
        be = self.be
        b, c = B.shape
        if self.world == 1 or b > c or not hasattr(be, "two_norm_gram"):
            return be.two_norm(B, rtol, max_iters)
        step = -(-c // self.world)
        step = -(-step // 16) * 16                      # K chunks on 16-column boundaries (TMA k-tiles)
        c0, c1 = min(c, self.rank * step), min(c, (self.rank + 1) * step)
        G = self._gbuf(b)
        G.zero_()
        if c1 > c0:
            be.gemm(GemmSpec(x=B, xm=0, y=B, yn=0, m=b, n=b, segs=[(c0, c0, c1 - c0)], c=G, lower=True,
                             mirror=True, tma_safe=True, xrows=b, xcols=c, yrows=b, ycols=c))
        self.comm.all_reduce(self._gb[:b])          # the contiguous b × ldg block (padding columns are zero)
        y1 = B.sum(dim=1) * (1.0 / float(np.sqrt(c)))
        return be.two_norm_gram(B, G, y1, rtol, max_iters)

    def _gbuf(self, b):
        buf = getattr(self, "_gb", None)
        ldg = -(-b // 32) * 32
        if buf is None or buf.shape[0] < b or buf.shape[1] != ldg:
            self._gb = buf = self.be.zeros(b, ldg)
        return buf[:b, :b]

    def sweep(self, rtol: float = 1e-9, max_iters: int = 5000):
        for k in range(len(self.ranges)):
            self.block_update(k)
        return self.error_estimate(len(self.ranges) - 1, rtol, max_iters)

    # ------------------------------------------------------------ residual / result
    def frobenius(self) -> float:
        """‖I − AΣ‖_F = ‖I − ΣA‖_F from local rows of ΣA, then all-reduce."""
        torch = self.torch
        part = torch.zeros(1, dtype=torch.float64, device=self.S.device)
        if self.operands == "sharded":
            # A's rows arrive chunk by chunk in natural order (all-gather of the row panels'
            # slices), so the δ of the fused epilogue sees contiguous global columns
            lay, be, p = self.layout, self.be, self.p
            chunk = lay.panel * self.world * max(1, 2048 // (lay.panel * self.world))
            for r0 in range(0, p, chunk):
                r1 = min(p, r0 + chunk)
                rows = self._gather_rows_natural(self.A, r0, r1)
                if self.n_loc:
                    part[0] += be.gemm(GemmSpec(x=self.S, xm=0, y=rows, yn=0, m=self.n_loc, n=r1 - r0,
                                                segs=[(0, 0, p)], cidx=self.own_t, cn=r0, frob=True, tma_safe=True,
                                                xrows=self.n_loc, xcols=p, yrows=r1 - r0, ycols=p))
        elif self.n_loc:
            v = self.be.gemm(GemmSpec(x=self.S, xm=0, y=self.A, yn=0, m=self.n_loc, n=self.p,
                                      segs=[(0, 0, self.p)], cidx=self.own_t, frob=True, tma_safe=True,
                                      xrows=self.n_loc, xcols=self.p, yrows=self.p, ycols=self.p))
            part[0] = v
        self.comm.all_reduce(part)
        return float(torch.sqrt(part)[0])

    def _gather_rows_natural(self, local, r0, r1):
        """Rows [r0, r1) of a row-panel-sharded matrix, natural order, on every rank."""
        lay, be = self.layout, self.be
        rng = [lay.local_range(h, r0, r1) for h in range(self.world)]
        nmax = max(1, max(b - a for a, b in rng))
        ld = local.stride(0) if local.shape[0] else self.ld
        key = (nmax, ld)
        if getattr(self, "_rowstage_key", None) != key:
            self._rowstage = be.zeros(self.world, nmax, ld)
            self._rownat = be.zeros(lay.panel * self.world * max(1, 2048 // (lay.panel * self.world)), ld)
            self._rowstage_key = key
        a, b = rng[self.rank]
        mine = be.zeros(nmax, ld)
        if b > a:
            mine[: b - a, : local.shape[1]] = local[a:b]
        self.comm.all_gather_start(self._rowstage, mine).wait()
        out = self._rownat[: r1 - r0]
        for h in range(self.world):
            a, b = rng[h]
            if b > a:
                out.index_copy_(0, self.rows_t[h][a:b] - r0, self._rowstage[h][: b - a])
        return out[:, : self.p]

    def gather_sigma(self):
        """Full Σ (host numpy) on every rank, original index order."""
        torch = self.torch
        counts = [len(r) for r in self.layout.rows]
        allrows = self.comm.all_gather_rows(self.S[: self.n_loc, : self.p], counts)
        order = np.concatenate(self.layout.rows)
        full = np.empty((self.p, self.p))
        if allrows.is_cuda and hasattr(self.be, "rows_to_host"):
            self.be.rows_to_host(allrows, full, order)     # panels land in their global rows directly
        else:
            full[order] = allrows.cpu().numpy()
        if self.perm is not None:
            inv = np.argsort(self.perm)
            full = full[np.ix_(inv, inv)]
        return full

    @staticmethod
    def comm_model(p: int, lo: int, hi: int, world: int, rank: int, panel: int = 128, operands: str = "sharded") -> dict:
        """The byte / flop model behind :meth:`comm_bytes`, from the layout alone (no process group):
        rank ``rank`` of ``world`` in the block step of set [lo, hi)."""
        lay = RowPanels(p, world, panel)
        b = hi - lo
        a0, a1 = lay.local_range(rank, lo, hi)
        n_loc = len(lay.rows[rank])
        n_I, n_cl, c = a1 - a0, n_loc - (a1 - a0), p - b
        return {"exchange_out": 8 * (b - n_I) * n_cl, "exchange_in": 8 * n_I * (c - n_cl),
                "allreduce_top": int(8 * b * b * 2 * (world - 1) / world),
                "allgather_w_in": 8 * b * (p - n_loc) if operands == "sharded" and world > 1 else 0,
                "gemm_flops": 2 * b * c * n_cl + 2 * b * b * n_cl}

    def comm_bytes(self, k: int) -> dict:
        """Bytes this rank moves over NVLink in block step k (each direction), by phase:
        the b × c transpose exchange (fused peer stores or all_to_all), the ring
        all-reduce of the b × b lower-triangle partials, and — operands sharded — the
        all-gather of W_k's column shards.  ``gemm_flops`` is this rank's share of
        2bc² + 2b²c, for the comm/compute budget in DESIGN.md §6."""
        pl = self.plan[k]
        return self.comm_model(self.p, pl["lo"], pl["hi"], self.world, self.rank, self.layout.panel, self.operands)

    def close(self):
        for work, _ in getattr(self, "_wpending", {}).values():
            work.wait()
        self._wpending = {}
        self.be.close()


# --------------------------------------------------------------------------- public entry point
def solve_sharded(a, part: Partition, cfg=None, *, group=None, panel: int = 128, device: int | None = None,
                  exchange: str = "auto", backend=None, gather_result: bool = True, callback=None,
                  operands: str = "auto", sigma0_cc=None):
    """``solve`` (reference solver.py:225-278) with Σ sharded over the process group.

    Call it on every rank with the same ``a`` (host array or a device copy) and
    partition.  Same loop and stop rules as the single-GPU ``solve``: K block
    updates, the reference's error estimate on the last set, stop when it is
    ≤ ``cfg.tol`` (``stopping="frobenius"``: ‖I − AΣ‖_F < tol, evaluated only
    once the estimate is below 1.01·tol, since ‖I − AΣ‖_F ≥ the estimate).
    Every rank returns the same trace; ``result`` is the full Σ (host numpy,
    original index order) on every rank when ``gather_result``, else None.
    Every reference guess is supported (identity / jacobi are seeded per panel; local, mc
    and takahashi are formed replicated by the single-GPU kernels, or passed as
    ``sigma0_cc``); FP64 DMMA GEMMs only.
    """
    import time
    import warnings

    from .exceptions import NoConvergenceWarning
    from .partition import validate
    from .solver import IbmiConfig, SolveReport

    cfg = cfg or IbmiConfig()
    if getattr(cfg, "gemm", None) == "ozaki":
        raise NotImplementedError("the sharded sweep runs FP64 DMMA GEMMs only (gemm='ozaki' is single-GPU)")
    validate(part)
    stopping = getattr(cfg, "stopping", "estimate")
    t0 = time.perf_counter()
    ss = ShardedSolver(a, part, group=group, panel=panel, backend=backend, device=device, exchange=exchange,
                       operands=operands)
    try:
        if sigma0_cc is None and cfg.initial_guess not in ("identity", "jacobi"):
            # local / mc / takahashi (solver.py:162-222): the single-GPU kernels form Σ₀[c₁,c₁] on
            # every rank from the same inputs (replicated, O(c³) once per solve)
            from .solver import make_initial_guess

            lo, hi = ss.ranges[0]
            if ss.perm is not None:
                raise NotImplementedError("non-trivial guesses with relabelled (non-contiguous) partitions")
            comp0 = np.concatenate([np.arange(0, lo), np.arange(hi, ss.p)])
            sigma0_cc = make_initial_guess(a, comp0, cfg)
        ss.init_sigma(cfg.initial_guess, sigma0_cc)
        setup_s = time.perf_counter() - t0
        errs, walls, pits, resid = [], [], [], []
        converged = False
        for _ in range(cfg.max_iterations):
            t1 = time.perf_counter()
            err, it, ok = ss.sweep(cfg.norm_rtol, cfg.norm_max_iters)
            if not ok:
                warnings.warn(f"two_norm: power iteration did not stabilize in {cfg.norm_max_iters} "
                              "iterations; returning last estimate", NoConvergenceWarning, stacklevel=2)
            fr = None
            if stopping == "frobenius":      # the same exact skip as the single-GPU loop (solver.run_solve)
                fr = ss.frobenius() if (getattr(cfg, "residual_every_sweep", False) or err < 1.01 * cfg.tol) \
                    else float("nan")
                resid.append(fr)
            walls.append(time.perf_counter() - t1)
            errs.append(err)
            pits.append(it)
            if callback is not None:
                callback(len(errs), err, fr)
            if (fr < cfg.tol) if fr is not None else (err <= cfg.tol):   # nan < tol is False
                converged = True
                break
        result = ss.gather_sigma() if gather_result else None
        return SolveReport(iterations=len(errs), converged=converged, error_trace=errs, wall_times=walls,
                           result=result, power_iterations=pits, residual_trace=resid, setup_seconds=setup_s)
    finally:
        ss.close()
