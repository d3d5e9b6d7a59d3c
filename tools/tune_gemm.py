"""Time the sweep's kernel classes under each GEMM path / variant / split-K factor."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_06377_b200 import _abi, configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

cfg = configs.get_config(sys.argv[1] if len(sys.argv) > 1 else "c4")
combos = [(0, 0, 0), (1, 0, 0), (1, 0, 1), (1, 0, 2), (1, 0, 3), (1, 0, 4)]   # (tma, variant, split)
a = torch.as_tensor(configs.make_matrix(cfg.name), device="cuda")
L = _abi.lib()
ds = DeviceSolver(a, partition=cfg.partition())
ds.setup()
ds.init_sigma(0)
s0 = ds.sigma(on_device=True)
ref = None
for tma, variant, split in combos:
    _abi.check(L.ibmi_tune(3, tma))
    _abi.check(L.ibmi_tune(0, variant))
    _abi.check(L.ibmi_tune(1, split))
    _abi.check(L.ibmi_tune(2, split))
    ds.set_sigma(s0)
    res = [ds.sweep_timed(1e-9, 5000) for _ in range(3)]
    t = {k: min(r[3][k] for r in res) for k in res[0][3]}
    ds.set_sigma(s0)
    ds.sweep_timed(1e-9, 5000)
    s1 = ds.sigma(on_device=True)
    if ref is None:
        ref = s1
    d = ((s1 - ref).norm() / ref.norm()).item()
    print(f"tma {tma} variant {variant} split {split}: " + " ".join(f"{k}={v:.2f}" for k, v in t.items()) +
          f"  err={res[-1][0]:.6e} dSigma={d:.1e}", flush=True)
fr = ds.frobenius()
_abi.check(L.ibmi_tune(3, 0))
fr0 = ds.frobenius()
print("frobenius tma / cp.async:", fr, fr0)
