"""Where does the end-to-end solve() time go? (c4, host buffers)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2502_06377_b200 as pkg  # noqa: E402
from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

cfg = configs.get_config("c4")
a = configs.make_matrix("c4")
part = cfg.partition()
torch.cuda.init()
for rep in range(2):
    T = {}
    t = time.perf_counter()
    ds = DeviceSolver(a, partition=part)
    torch.cuda.synchronize(); T["create+upload"] = time.perf_counter() - t; t = time.perf_counter()
    ds.setup()
    T["setup"] = time.perf_counter() - t; t = time.perf_counter()
    ds.init_sigma(0)
    T["init"] = time.perf_counter() - t; t = time.perf_counter()
    ds.sweep(1e-9, 5000)
    T["first sweep (capture)"] = time.perf_counter() - t; t = time.perf_counter()
    for _ in range(9):
        ds.sweep(1e-9, 5000)
    T["9 sweeps"] = time.perf_counter() - t; t = time.perf_counter()
    s = ds.sigma()
    T["download"] = time.perf_counter() - t; t = time.perf_counter()
    ds.close()
    T["close"] = time.perf_counter() - t
    print(rep, {k: round(v, 3) for k, v in T.items()}, flush=True)
t = time.perf_counter()
rep = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-300, max_iterations=10))
print("solve() 10 sweeps:", round(time.perf_counter() - t, 3))
os.environ["IBMI_PROFILE"] = "1"
for _ in range(2):
    t = time.perf_counter()
    rep = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-300, max_iterations=10))
    print("solve() 10 sweeps:", round(time.perf_counter() - t, 3), flush=True)
    del rep
