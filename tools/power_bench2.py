"""Power-iteration device time per iteration inside real sweeps (c1..c4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

for name in sys.argv[1:]:
    cfg = configs.get_config(name)
    a = torch.as_tensor(configs.make_matrix(name), device="cuda")
    ds = DeviceSolver(a, partition=cfg.partition())
    ds.setup()
    ds.init_sigma(1 if cfg.guess == "jacobi" else 0)
    tot_ms, tot_it = 0.0, 0
    for _ in range(6):
        e, it, cv, t = ds.sweep_timed(1e-9, 5000)
        tot_ms += t["power_iteration"]
        tot_it += it
    print(f"{name}: {tot_it} iterations, {tot_ms:.3f} ms, {tot_ms / tot_it * 1e3:.2f} us/iter; last sweep {t}", flush=True)
    ds.close()
