"""Graph-replayed vs eagerly launched sweeps in one process (device time per
sweep, SM clock sampled during each phase).  usage: moduli sweeps [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402
from bench import ClockSampler  # noqa: E402

moduli = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
name = sys.argv[3] if len(sys.argv) > 3 else "c4"
cfg = configs.get_config(name)
a = torch.as_tensor(configs.make_matrix(name), device="cuda")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
ds = DeviceSolver(a, partition=cfg.partition(), stream=stream.cuda_stream)
ds.set_emulation(moduli)
ds.setup()
ds.init_sigma(1 if cfg.guess == "jacobi" else 0)
for _ in range(3):
    ds.sweep(1e-9, 5000)
torch.cuda.synchronize()


def timed(label, fn):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        for _ in range(n):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
    print(f"{label}: {e0.elapsed_time(e1) / n:.2f} ms/sweep, clocks {clk.summary()}", flush=True)


for rep in range(2):
    timed("graph", lambda: ds.sweep(1e-9, 5000))
    timed("eager (sweep_timed)", lambda: ds.sweep_timed(1e-9, 5000))
