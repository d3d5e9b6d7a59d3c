"""Sweep kernel-class times under each FP64 GEMM tile raster (ibmi_tune key 12),
from the same Σ each time; prints the Σ difference against the first setting."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_06377_b200 import _abi, configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

cfg = configs.get_config(sys.argv[1] if len(sys.argv) > 1 else "c4")
groups = [int(g) for g in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 4, 8, 16]
a = torch.as_tensor(configs.make_matrix(cfg.name), device="cuda")
L = _abi.lib()
ds = DeviceSolver(a, partition=cfg.partition())
ds.setup()
ds.init_sigma(1 if cfg.guess == "jacobi" else 0)
ds.sweep(1e-9, 5000)
s0 = ds.sigma(on_device=True).clone()
ref = None
for rep in range(2):
    for g in groups:
        _abi.check(L.ibmi_tune(12, g))
        ds.set_sigma(s0)
        res = [ds.sweep_timed(1e-9, 5000) for _ in range(3)]
        t = {k: min(r[3][k] for r in res) for k in res[0][3]}
        ds.set_sigma(s0)
        ds.sweep(1e-9, 5000)
        s1 = ds.sigma(on_device=True)
        if ref is None:
            ref = s1.clone()
        d = float((s1 - ref).norm() / ref.norm())
        print(f"{cfg.name} group {g:3d}: " + " ".join(f"{k}={v:.3f}" for k, v in t.items()) + f" dSigma={d:.1e}",
              flush=True)
ds.close()
