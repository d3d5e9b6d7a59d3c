"""Print the error / residual trajectory of a BASELINE config on the GPU."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2])
every = int(sys.argv[3]) if len(sys.argv) > 3 else 10
moduli = int(sys.argv[4]) if len(sys.argv) > 4 else 0   # 0: FP64 DMMA, else Ozaki-II moduli
cfg = configs.get_config(name)
a = torch.as_tensor(configs.make_matrix(name), device="cuda")
ds = DeviceSolver(a, partition=cfg.partition())
if moduli:
    ds.set_emulation(moduli)
t0 = time.perf_counter()
ds.setup()
ds.init_sigma(1 if cfg.guess == "jacobi" else 0)
for it in range(1, n + 1):
    e, pi, conv = ds.sweep(1e-9, 5000)
    if it % every == 0 or it <= 5:
        fr = ds.frobenius()
        print(f"sweep {it} err {e:.4e} pit {pi} frob {fr:.4e} t={time.perf_counter() - t0:.1f}s", flush=True)
