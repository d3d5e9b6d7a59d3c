"""Profiling driver for the sharded sweep at world size 1 (NCCL): construct,
Σ₀, one warm-up sweep, then ONE sweep between cudaProfilerStart/Stop, with a
CUDA-event phase breakdown of that sweep.  Use with ncu --profile-from-start off."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.distributed import ShardedSolver  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4")
ap.add_argument("--exchange", default="auto")
ap.add_argument("--sweeps", type=int, default=3)
ap.add_argument("--operands", default="auto")
args = ap.parse_args()
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29541")
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
cfg = configs.get_config(args.config)
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
a = torch.as_tensor(configs.make_matrix(args.config), device="cuda")
ss = ShardedSolver(a, cfg.partition(), exchange=args.exchange, operands=args.operands)
print("operands", ss.operands, "exchange", ss.exchange, flush=True)
ss.init_sigma(cfg.guess if cfg.guess in ("identity", "jacobi") else "identity")
ss.sweep()
torch.cuda.synchronize()
for i in range(args.sweeps):
    t = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    ss.sweep()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"sweep {i}: wall {1e3 * (time.perf_counter() - t):.2f} ms, device {e0.elapsed_time(e1):.2f} ms", flush=True)
torch.cuda.profiler.start()
ss.sweep()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ss.close()
dist.destroy_process_group()
