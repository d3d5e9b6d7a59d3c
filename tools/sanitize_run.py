"""Small end-to-end workload touching every kernel path, for compute-sanitizer."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import paper_2502_06377_b200 as pkg  # noqa: E402
from conftest import random_spd  # noqa: E402
from paper_2502_06377_b200 import linalg  # noqa: E402

for p, k, f in [(9, 4, 0.0), (300, 3, 0.1), (520, 4, 0.125), (1100, 3, 0.2)]:
    a = random_spd(p, p)
    rep = pkg.solve(a, pkg.contiguous_partition(p, k, f), pkg.IbmiConfig(tol=1e-300, max_iterations=2))
    rep = pkg.solve(a, pkg.contiguous_partition(p, k, f), pkg.IbmiConfig(tol=1e-10, max_iterations=2,
                                                                      stopping="frobenius", initial_guess="jacobi"))
a = random_spd(256, 3)
pkg.solve(a, pkg.red_black_partition(256), pkg.IbmiConfig(tol=1e-300, max_iterations=2, initial_guess="takahashi"))
perm = np.random.default_rng(1).permutation(256)
part = pkg.load_partition_json({"p": 256, "sets": [np.sort(perm[:150]).tolist(), np.sort(perm[120:]).tolist()]})
pkg.solve(a, part, pkg.IbmiConfig(tol=1e-300, max_iterations=2, initial_guess="mc", mc_samples=20))
linalg.spd_inverse(random_spd(200, 4))
linalg.two_norm(np.random.default_rng(0).standard_normal((700, 900)))
linalg.two_norm(np.random.default_rng(1).standard_normal((1300, 800)))       # column-Gram form, flag-exchange kernel
# the sharded driver's kernels (ibmi_gemm descriptors, ibmi_sym_rows) at world size 1, both operand modes
import torch.distributed as dist  # noqa: E402

from paper_2502_06377_b200.distributed import ShardedSolver  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29577")
dist.init_process_group("gloo", rank=0, world_size=1)
for operands in ("replicated", "sharded"):
    a = random_spd(520, 5)
    ss = ShardedSolver(a, pkg.contiguous_partition(520, 4, 0.125), panel=64, device=0, exchange="nccl",
                       operands=operands)
    ss.init_sigma("jacobi")
    ss.sweep()
    ss.frobenius()
    ss.close()
dist.destroy_process_group()
print("sanitize workload done")
