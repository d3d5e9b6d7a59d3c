"""Second floor probe: which stage of the GPU SPD inverse sets the c4 floor?

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
    install(ours, "ours (blocked potrf + trtri + L^-T L^-1)")
    tl = [torch.linalg.cholesky(b) for b in blocks]
    install([sym(torch.cholesky_solve(eye(len(b)), l)) for b, l in zip(blocks, tl)], "library chol + library potrs(I)")
    install([sym(torch.cholesky_inverse(l)) for l in tl], "library chol + library potri")
    ol = [linalg.cholesky(b).l for b in blocks]
    print("our L vs library L:", [f"{float(torch.linalg.norm(o - t) / torch.linalg.norm(t)):.1e}" for o, t in zip(ol, tl)][:3])
    install([sym(torch.cholesky_solve(eye(len(b)), l)) for b, l in zip(blocks, ol)], "our chol + library potrs(I)")
    install([sym(torch.cholesky_inverse(l)) for l in ol], "our chol + library potri")
    li = [torch.linalg.solve_triangular(l, eye(len(l)), upper=False) for l in tl]
    install([sym(x.T @ x) for x in li], "library chol + library trtri + product")
    install([sym(x + x @ (eye(len(b)) - b @ x)) for x, b in zip(ours, blocks)], "ours + one Newton step")
    install([sym(x + (eye(len(b)) - x @ b) @ x) for x, b in zip(ours, blocks)], "ours + one left Newton step")
