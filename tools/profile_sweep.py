"""Profiling driver: set up a BASELINE config, warm up, then run ONE sweep
(no graph, so every kernel is a separate launch) between
cudaProfilerStart/Stop.  Use with ncu --profile-from-start off."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--sweeps", type=int, default=1)
ap.add_argument("--tune", action="append", default=[], help="key=value for ibmi_tune (repeatable)")
args = ap.parse_args()
if args.tune:
    from paper_2502_06377_b200 import _abi

    for kv in args.tune:
        k, v = kv.split("=")
        _abi.check(_abi.lib().ibmi_tune(int(k), int(v)), "tune")
cfg = configs.get_config(args.config)
a = torch.as_tensor(configs.make_matrix(args.config), device="cuda")
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
ds = DeviceSolver(a, partition=cfg.partition(), stream=s.cuda_stream)
ds.setup()
ds.init_sigma(1 if cfg.guess == "jacobi" else 0)
ds.sweep_timed(1e-9, 5000)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(args.sweeps):
    err, it, conv, t = ds.sweep_timed(1e-9, 5000)
    print(f"power iterations {it}: {t['power_iteration'] * 1e3:.1f} us", flush=True)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("sweep ms", t)
