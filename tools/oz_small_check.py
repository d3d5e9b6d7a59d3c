import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2502_06377_b200 as pkg
from paper_2502_06377_b200.device import DeviceSolver
p = int(sys.argv[1]) if len(sys.argv) > 1 else 3072
m = np.random.default_rng(0).standard_normal((p, p)); a = m.T @ m + p * np.eye(p)
part = pkg.contiguous_partition(p, 4, 0.125)
r0 = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-11, gemm="dmma"))
r1 = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-11, gemm="ozaki"))
print("iters", r0.iterations, r1.iterations, "rel", np.linalg.norm(r1.result - r0.result) / np.linalg.norm(r0.result))
with DeviceSolver(a, partition=part) as ds:
    ds.set_emulation(16); ds.setup(); ds.init_sigma(0)
    print(ds.sweep_timed(1e-9, 5000))
    torch.cuda.synchronize()
