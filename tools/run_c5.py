"""c5 (p=65536, 16 sets) on one B200: generate A on the device, set up, run N sweeps."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
moduli = int(sys.argv[2]) if len(sys.argv) > 2 else 0      # 0: FP64 DMMA, 8..20: Ozaki-II emulation
cfg = configs.get_config("c5")
t0 = time.perf_counter()
a = configs.make_matrix_c5_device(0)
torch.cuda.synchronize()
print(f"generated A in {time.perf_counter() - t0:.1f}s; mem {torch.cuda.memory_allocated() / 1e9:.1f} GB", flush=True)
ds = DeviceSolver(a, partition=cfg.partition())
del a
torch.cuda.empty_cache()
ds.set_emulation(moduli)
t0 = time.perf_counter()
ds.setup()
ds.init_sigma(0)
torch.cuda.synchronize()
print(f"setup {time.perf_counter() - t0:.2f}s; context bytes {ds.device_bytes() / 1e9:.1f} GB", flush=True)
fl = configs.sweep_flops(cfg)
t_run = time.perf_counter()
for it in range(n):
    e, pi, cv, t = ds.sweep_timed(1e-9, 5000)
    if e <= cfg.tol:
        print(f"converged after {it + 1} sweeps: err {e:.4e} <= tol {cfg.tol}; sweeps wall {time.perf_counter() - t_run:.1f}s", flush=True)
    print(f"sweep {it + 1} err {e:.4e} pit {pi} ms {t['sweep']:.0f} -> {fl / t['sweep'] / 1e9:.2f} TF/s {t}", flush=True)
