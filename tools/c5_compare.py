"""c5 (p=65536): FP64 DMMA vs Ozaki-II emulation after the same sweeps from the
same Σ0 — sampled rows, row sums and ‖Σ‖_F (Σ itself is 34 GB)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

nsweeps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = configs.get_config("c5")
rows = np.sort(np.random.default_rng(5).choice(cfg.p, 64, replace=False))
out = {}
for mode in (0, 16):
    a = configs.make_matrix_c5_device(0)
    torch.cuda.synchronize()
    ds = DeviceSolver(a, partition=cfg.partition())
    del a
    torch.cuda.empty_cache()
    ds.set_emulation(mode)
    t0 = time.perf_counter()
    ds.setup()
    ds.init_sigma(0)
    errs = []
    for _ in range(nsweeps):
        errs.append(ds.sweep(1e-9, 5000)[0])
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ds.set_emulation(0)          # releases the residue caches (Σ unchanged) to make room for the copy
    s = ds.sigma(on_device=True)
    samp = s[torch.as_tensor(rows, device=s.device)].cpu().numpy()
    rs = s.sum(dim=1).cpu().numpy()
    fro = float(torch.linalg.norm(s))
    del s
    ds.close()
    torch.cuda.empty_cache()
    out[mode] = (errs, samp, rs, fro)
    print(f"moduli={mode}: {dt:.1f}s setup+{nsweeps} sweeps, errs {['%.6e' % e for e in errs]}, |Sigma|_F {fro:.12e}",
          flush=True)
e0, s0, r0, f0 = out[0]
e1, s1, r1, f1 = out[16]
print(f"sampled rows rel-fro {np.linalg.norm(s1 - s0) / np.linalg.norm(s0):.3e}; "
      f"row sums rel {np.linalg.norm(r1 - r0) / np.linalg.norm(r0):.3e}; "
      f"|Sigma|_F rel {abs(f1 - f0) / f0:.3e}; err trace max rel {max(abs(x - y) / y for x, y in zip(e1, e0)):.3e}",
      flush=True)
