"""Phase timings of repeated solve() calls on host buffers (IBMI_PROFILE=1, device-synchronised)."""
import os
import sys
import time

os.environ["IBMI_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_06377_b200 as pkg  # noqa: E402
from paper_2502_06377_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = configs.get_config(name)
a = configs.make_matrix(name)
part = cfg.partition()
for r in range(reps):
    t = time.perf_counter()
    rep = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-300, max_iterations=10))
    print(f"rep {r}: solve() 10 sweeps {time.perf_counter() - t:.3f}s", file=sys.stderr, flush=True)
    del rep
