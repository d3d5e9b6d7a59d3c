"""Stress the flag-exchange power iteration (power_gram_ll_kernel): the tagged 128-byte line must
never be seen torn.  A torn read would change σ or the iteration count, so every repetition of
two_norm on the same matrix must return bit-identical σ and the same count; also against the
grid-barrier kernel (ibmi_tune key 13 = 0), whose σ agrees to ~1e-15.

usage: python tools/ll_determinism_stress.py [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_06377_b200 import _abi  # noqa: E402
from paper_2502_06377_b200.linalg import two_norm  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
bad = 0
for shape, seed in [((2048, 2048), 1), ((1152, 7040), 2), ((2200, 2600), 3), ((700, 1500), 4), ((1536, 900), 5)]:
    rng = np.random.default_rng(seed)
    b = torch.as_tensor(rng.standard_normal(shape) * np.exp(rng.uniform(-1, 1, size=(shape[0], 1))), device="cuda")
    s0 = two_norm(b)
    it0 = two_norm.last_iterations
    t = time.perf_counter()
    n_bad = 0
    for _ in range(reps):
        s = two_norm(b)
        if s != s0 or two_norm.last_iterations != it0:
            n_bad += 1
    dt = time.perf_counter() - t
    _abi.check(_abi.lib().ibmi_tune(13, 0), "tune")
    sb = two_norm(b)
    itb = two_norm.last_iterations
    _abi.check(_abi.lib().ibmi_tune(13, 1), "tune")
    print(f"{shape}: sigma {s0:.15e} iterations {it0}; {reps} repetitions, {n_bad} differing, {dt / reps * 1e3:.2f} ms each; "
          f"barrier kernel: rel diff {abs(sb - s0) / s0:.1e}, iterations {itb}", flush=True)
    bad += n_bad
print("TORN OR NONDETERMINISTIC READS:" if bad else "all repetitions bit-identical:", bad)
sys.exit(1 if bad else 0)
