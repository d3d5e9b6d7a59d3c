"""Phase timings of distributed.solve_sharded pieces on one rank (NCCL world 1 by default,
or under torchrun): solver construction (A upload + setup), Σ₀, sweeps, Σ gather to host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.distributed import ShardedSolver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
os.environ.setdefault("RANK", "0")
os.environ.setdefault("WORLD_SIZE", "1")
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
cfg = configs.get_config(name)
a = configs.make_matrix(name)
part = cfg.partition()
for rep in range(2):
    T = {}
    dist.barrier()
    t = time.perf_counter()
    ss = ShardedSolver(a, part)
    torch.cuda.synchronize()
    T["construct"] = time.perf_counter() - t
    t = time.perf_counter()
    ss.init_sigma(cfg.guess if cfg.guess in ("identity", "jacobi") else "identity")
    torch.cuda.synchronize()
    T["init"] = time.perf_counter() - t
    for i in range(3):
        t = time.perf_counter()
        ss.sweep()
        torch.cuda.synchronize()
        T[f"sweep{i}"] = time.perf_counter() - t
    t = time.perf_counter()
    full = ss.gather_sigma()
    T["gather"] = time.perf_counter() - t
    t = time.perf_counter()
    ss.close()
    T["close"] = time.perf_counter() - t
    if dist.get_rank() == 0:
        print(name, rep, {k: round(v, 4) for k, v in T.items()}, flush=True)
    del full
dist.destroy_process_group()
