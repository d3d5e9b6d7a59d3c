import sys, time, os
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2502_06377_b200 as pkg
from paper_2502_06377_b200 import configs
cfg = configs.get_config("c4")
a = configs.make_matrix("c4")
part = cfg.partition()
for gemm in ("ozaki", "dmma", "ozaki"):
    for it in range(2):
        t0 = time.perf_counter()
        rep = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-300, max_iterations=10, gemm=gemm))
        print(gemm, f"wall {time.perf_counter() - t0:.3f}s setup {rep.setup_seconds:.3f} sweeps {sum(rep.wall_times):.3f}", flush=True)
