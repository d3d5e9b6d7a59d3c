"""CPU emulation of the sharded solver's compute backend — TEST DOUBLE ONLY.

Implements the GemmSpec semantics of paper_2502_06377_b200.distributed (and
include/ibmi_b200.h::ibmi_gemm) with torch CPU float64 ops, so the
multi-process exchange logic can be exercised with the gloo backend on hosts
without a GPU.  The product never imports this module.
"""

import numpy as np
import torch

from oracle import ibmi_oracle as orc
from paper_2502_06377_b200.distributed import GemmSpec, map_indices


class TorchCPUBackend:
    def __init__(self):
        self.device = torch.device("cpu")

    def setup(self, a, ranges):
        a = np.asarray(a, dtype=np.float64)
        p = a.shape[0]
        A = torch.as_tensor(a.copy())
        W, ainv = [], []
        for lo, hi in ranges:
            inv = orc.spd_inverse(a[lo:hi, lo:hi])
            w = inv @ a[lo:hi, :]
            w[:, lo:hi] = 0.0
            W.append(torch.as_tensor(w))
            ainv.append(torch.as_tensor(inv))
        return A, W, ainv

    def upload_rows(self, a, rows):
        return torch.as_tensor(np.asarray(a, dtype=np.float64)[np.asarray(rows, dtype=np.int64), :].copy())

    def transposed(self, t):
        return t.t().contiguous()

    def spd_inverse(self, blk):
        return torch.as_tensor(orc.spd_inverse(np.asarray(blk, dtype=np.float64)))

    def sym_rows(self, base, low, rel, dst):
        full = torch.tril(low) + torch.tril(low, -1).T
        dst.copy_(base[rel] + full[rel])

    def zeros(self, *shape):
        return torch.zeros(shape, dtype=torch.float64)

    def index_tensor(self, idx):
        return torch.as_tensor(np.asarray(idx, dtype=np.int64))

    def gemm(self, s: GemmSpec):
        rx = torch.as_tensor(map_indices(s.xm, s.m))
        ry = torch.as_tensor(map_indices(s.yn, s.n))
        acc = torch.zeros((s.m, s.n), dtype=torch.float64)
        for x0, y0, ln in s.segs:
            if ln > 0:
                xs = s.x[x0:x0 + ln][:, rx].T if s.xt else s.x[rx, x0:x0 + ln]
                ys = s.y[y0:y0 + ln][:, ry].T if s.yt else s.y[ry, y0:y0 + ln]
                acc += xs @ ys.T
        crow = s.cidx if s.cidx is not None else torch.as_tensor(map_indices(s.cm, s.m))
        ccol = torch.as_tensor(map_indices(s.cn, s.n))
        if s.frob:
            delta = (crow[:, None] == ccol[None, :]).to(torch.float64)
            return ((delta - acc) ** 2).sum()
        v = s.alpha * acc
        if s.beta != 0.0:
            v = v + s.beta * s.d[torch.as_tensor(map_indices(s.dm, s.m))][:, torch.as_tensor(map_indices(s.dn, s.n))]
        keep = torch.ones_like(v, dtype=torch.bool)
        if s.lower:
            keep = torch.tril(keep)
        if s.direct:
            mi, ni = torch.nonzero(keep, as_tuple=True)
            s.c[crow[mi], ccol[ni]] = v[mi, ni]
        if s.mirror:
            c2 = s.c2 if s.c2 is not None else s.c
            c2m = torch.as_tensor(map_indices(s.c2m if s.c2 is not None else s.cm, s.m))
            c2n = torch.as_tensor(map_indices(s.c2n if s.c2 is not None else s.cn, s.n))
            mi, ni = torch.nonzero(keep, as_tuple=True)
            c2[c2n[ni], c2m[mi]] = v[mi, ni]
        return None

    def gemm_xt(self, x, x_col0, y, m, n, segs, c, alpha=1.0):
        acc = torch.zeros((m, n), dtype=torch.float64)
        for x0, y0, ln in segs:
            if ln > 0:
                acc += x[x0:x0 + ln, x_col0:x_col0 + m].T @ y[:n, y0:y0 + ln].T
        c[:m, :n] = alpha * acc

    def two_norm(self, b, rtol, max_iters):
        s, conv, it = orc.power_sigma_max(b.numpy(), rtol, max_iters)
        return s, it, conv

    def two_norm_gram(self, b, g, y1, rtol, max_iters):
        # the caller's Gram matrix and y1 must be what the library would have formed itself
        bn = b.numpy()
        assert np.allclose(g.numpy(), bn @ bn.T, rtol=1e-10, atol=1e-10 * float(np.abs(g.numpy()).max() + 1e-300))
        assert np.allclose(y1.numpy(), bn.sum(axis=1) / np.sqrt(bn.shape[1]), rtol=1e-10, atol=1e-12)
        s, conv, it = orc.power_sigma_max(bn, rtol, max_iters)
        return s, it, conv

    def close(self):
        pass
