"""Third floor probe (candidate fixes, emulated with torch on the GPU).

Second floor probe: which stage of the GPU SPD inverse sets the c4 floor?

Every variant writes its A_II⁻¹ (and W = A_II⁻¹·A_Ic by a library GEMM) into the
context's buffers and runs the same GPU sweeps.  Variants: library potrs / potri on
library or our Cholesky factor, our inverse, our inverse after one Newton step.

usage: python tools/c4_floor_probe2.py [config] [sweeps]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_06377_b200 import _abi, configs, linalg  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
nsweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cfg = configs.get_config(name)
a = configs.make_matrix(name)
part = cfg.partition()
p = cfg.p
L = _abi.lib()


def view(ds, which, k=0):
    ptr, r, c, ld = C.c_void_p(), C.c_int64(), C.c_int64(), C.c_int64()
    _abi.check(L.ibmi_export(ds._h, which, k, C.byref(ptr), C.byref(r), C.byref(c), C.byref(ld)), "export")

    class V:
        __cuda_array_interface__ = {"shape": (int(r.value), int(c.value)), "typestr": "<f8",
                                    "data": (int(ptr.value), False), "strides": (int(ld.value) * 8, 8), "version": 3}
    return torch.as_tensor(V(), device="cuda")


def run(ds, tag):
    ds.init_sigma(1 if cfg.guess == "jacobi" else 0)
    errs = [ds.sweep(1e-9, 5000)[0] for _ in range(nsweeps)]
    print(f"{tag:44s} floor {min(errs):.3e} last {errs[-1]:.3e} frob {ds.frobenius():.4e}", flush=True)


def sym(x):
    return 0.5 * (x + x.T)


with DeviceSolver(a, partition=part) as ds:
    ds.setup()
    torch.cuda.synchronize()
    a_dev = torch.as_tensor(a, device="cuda")
    rng = [(int(i[0]), int(i[-1]) + 1) for i in part.sets]
    ours = [view(ds, 3, k)[:, : hi - lo].clone() for k, (lo, hi) in enumerate(rng)]
    eye = lambda n: torch.eye(n, dtype=torch.float64, device="cuda")   # noqa: E731

    def install(invs, tag):
        for k, (lo, hi) in enumerate(rng):
            view(ds, 3, k)[:, : hi - lo] = invs[k]
            wn = invs[k] @ a_dev[lo:hi, :]
            wn[:, lo:hi] = 0.0
            view(ds, 2, k)[:, :p] = wn
        torch.cuda.synchronize()
        run(ds, tag)

    blocks = [a_dev[lo:hi, lo:hi].contiguous() for lo, hi in rng]
    ol = [linalg.cholesky(b).l for b in blocks]
    NB = 64

    def leaf_inv(l):
        return torch.linalg.solve_triangular(l, eye(len(l)), upper=False)

    def rec_lower(l, b):          # solve l x = b
        n = len(l)
        if n <= NB:
            return leaf_inv(l) @ b
        h = (n // 2 + NB - 1) // NB * NB
        x1 = rec_lower(l[:h, :h], b[:h])
        x2 = rec_lower(l[h:, h:], b[h:] - l[h:, :h] @ x1)
        return torch.cat([x1, x2], 0)

    def rec_lower_t(l, b):        # solve l^T x = b
        n = len(l)
        if n <= NB:
            return leaf_inv(l).T @ b
        h = (n // 2 + NB - 1) // NB * NB
        x2 = rec_lower_t(l[h:, h:], b[h:])
        x1 = rec_lower_t(l[:h, :h], b[:h] - l[h:, :h].T @ x2)
        return torch.cat([x1, x2], 0)

    def our_trtri(l):
        n = len(l)
        x = l.clone()
        for j0 in range(((n - 1) // NB) * NB, -1, -NB):
            j1 = min(n, j0 + NB)
            d = leaf_inv(l[j0:j1, j0:j1])
            if j1 < n:
                x[j1:, j0:j1] = -(x[j1:, j1:] @ l[j1:, j0:j1]) @ d
            x[j0:j1, j0:j1] = d
        return x

    ys = [our_trtri(l) for l in ol]
    install([sym(y.T @ y) for y in ys], "emulated ours (our chol, blocked trtri, product)")
    install([sym(rec_lower_t(l, y)) for l, y in zip(ol, ys)], "C3: blocked trtri Y, recursive back-substitution")
    yr = [rec_lower(l, eye(len(l))) for l in ol]
    install([sym(rec_lower_t(l, y)) for l, y in zip(ol, yr)], "C1: recursive TRSM both steps (leaf 64)")
    install([sym(y.T @ y) for y in yr], "C4: recursive-TRSM Y, product")
    NB = 128
    yr = [rec_lower(l, eye(len(l))) for l in ol]
    install([sym(rec_lower_t(l, y)) for l, y in zip(ol, yr)], "C1 with leaf 128")
    NB = 64
    # C6: solve only the lower triangle of X (symmetric), block rows bottom-up
    def backsub_lower(l, y):
        n = len(l)
        x = torch.zeros_like(l)
        for j0 in range(((n - 1) // NB) * NB, -1, -NB):
            j1 = min(n, j0 + NB)
            t = y[j0:j1, :j1] - l[j1:, j0:j1].T @ x[j1:, :j1]
            x[j0:j1, :j1] = leaf_inv(l[j0:j1, j0:j1]).T @ t
            x[:j0, j0:j1] = x[j0:j1, :j0].T
        return x
    install([backsub_lower(l, y) for l, y in zip(ol, yr)], "C6: recursive Y, block-row back-substitution (lower, mirrored)")
