"""Sweep time vs the split-K minimum k-tiles per slice (small configs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_06377_b200 import _abi, configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

L = _abi.lib()
for name in sys.argv[1:]:
    cfg = configs.get_config(name)
    a = torch.as_tensor(configs.make_matrix(name), device="cuda")
    ds = DeviceSolver(a, partition=cfg.partition())
    ds.setup()
    ds.init_sigma(1 if cfg.guess == "jacobi" else 0)
    for _ in range(3):
        ds.sweep(1e-9, 5000)
    s0 = ds.sigma(on_device=True)
    for mkt in (8, 4, 2, 1):
        _abi.check(L.ibmi_tune(6, mkt))
        ds.set_sigma(s0)
        res = [ds.sweep_timed(1e-9, 5000)[3] for _ in range(3)]
        t = {k: min(r[k] for r in res) for k in res[0]}
        ds.set_sigma(s0)
        import time
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(20):
            ds.sweep(1e-9, 5000)
        wall = (time.perf_counter() - t0) / 20
        print(name, "min_kt", mkt, " ".join(f"{k}={v:.3f}" for k, v in t.items()), f"graph-sweep wall={wall*1e3:.3f}ms", flush=True)
    _abi.check(L.ibmi_tune(6, 4))
    ds.close()
