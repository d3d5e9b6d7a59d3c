"""Panel/estimate split-K on vs off, per config."""
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
    s0 = ds.sigma(on_device=True)
    ref = None
    for split in (1, 0, 2, 3):
        _abi.check(L.ibmi_tune(4, split))
        ds.set_sigma(s0)
        res = [ds.sweep_timed(1e-9, 5000) for _ in range(3)]
        t = {k: min(r[3][k] for r in res) for k in res[0][3]}
        ds.set_sigma(s0)
        ds.sweep_timed(1e-9, 5000)
        s1 = ds.sigma(on_device=True)
        ref = s1 if ref is None else ref
        print(name, "panel split", split, " ".join(f"{k}={v:.3f}" for k, v in t.items()),
              f"dSigma={((s1 - ref).norm() / ref.norm()).item():.1e}", flush=True)
    _abi.check(L.ibmi_tune(4, 0))
    ds.close()
    del a
    torch.cuda.empty_cache()
