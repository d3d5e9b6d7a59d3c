"""Profiling driver for ibmi_setup: a warm-up context, then ONE setup of a
second context between cudaProfilerStart/Stop (use with ncu --profile-from-start off)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--tune", action="append", default=[], help="key=value for ibmi_tune (repeatable)")
ap.add_argument("--reps", type=int, default=4)
args = ap.parse_args()
if args.tune:
    from paper_2502_06377_b200 import _abi

    for kv in args.tune:
        k, v = kv.split("=")
        _abi.check(_abi.lib().ibmi_tune(int(k), int(v)), "tune")
cfg = configs.get_config(args.config)
a = torch.as_tensor(configs.make_matrix(args.config), device="cuda")
for rep in range(args.reps):
    ds = DeviceSolver(a, partition=cfg.partition())
    torch.cuda.synchronize()
    if rep == args.reps - 1:
        torch.cuda.profiler.start()
    t = time.perf_counter()
    ds.setup()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    if rep == args.reps - 1:
        torch.cuda.profiler.stop()
    print(f"{args.config} setup {dt * 1e3:.1f} ms", flush=True)
    ds.close()
