"""µs per power iteration of ibmi_two_norm for Gram sizes of the configs."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2502_06377_b200.linalg import two_norm  # noqa: E402

for rows, cols in [(256, 256), (2048, 2048), (1152, 7040), (2304, 14080)]:
    g = torch.Generator(device="cuda").manual_seed(0)
    b = torch.randn((rows, cols), dtype=torch.float64, device="cuda", generator=g)
    b[:, 0] *= 1.05          # a mild gap: many iterations
    two_norm(b, 1e-12, 400)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = two_norm(b, 1e-300, 400)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{rows}x{cols}: {two_norm.last_iterations} iters, {dt * 1e3:.2f} ms total, "
          f"{dt / two_norm.last_iterations * 1e6:.2f} us/iter (incl. Gram GEMM)", flush=True)
