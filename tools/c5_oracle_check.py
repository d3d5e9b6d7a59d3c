"""c5 (p=65536) parity against the CPU oracle at full size: the first sweep.

The GPU runs setup + one sweep (16 block updates + the error estimate on the
last set) through the C ABI; the oracle (reference algorithm on NumPy/OpenBLAS,
test infrastructure) runs the same sweep from the same A and Σ₀ = I on the
host cores.  Σ is compared in row chunks (relative Frobenius), plus the error
estimate.  Needs ~140 GB of host RAM and ~20 min of CPU on the GPU box, so it
is a tool (log kept under profiles/), not a pytest case.

usage: python tools/c5_oracle_check.py [moduli]   (0 = FP64 DMMA, default)
"""
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import ibmi_oracle as orc  # noqa: E402
from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

moduli = int(sys.argv[1]) if len(sys.argv) > 1 else 0
cfg = configs.get_config("c5")
part = cfg.partition()
p = cfg.p
t0 = time.perf_counter()
a_dev = configs.make_matrix_c5_device(0)
a = a_dev.cpu().numpy()
print(f"A generated on the GPU and copied to the host in {time.perf_counter() - t0:.1f}s "
      f"(host cores {os.cpu_count()}, OPENBLAS_NUM_THREADS={os.environ['OPENBLAS_NUM_THREADS']})", flush=True)

# ---- GPU: setup + one sweep
ds = DeviceSolver(a_dev, partition=part)
del a_dev
torch.cuda.empty_cache()
if moduli:
    ds.set_emulation(moduli)
torch.cuda.synchronize()
t1 = time.perf_counter()
ds.setup()
ds.init_sigma(0)
err_gpu, pit_gpu, _ = ds.sweep(1e-9, 5000)
torch.cuda.synchronize()
print(f"GPU (moduli={moduli}): setup + 1 sweep {time.perf_counter() - t1:.1f}s, err {err_gpu:.12e}, "
      f"power iterations {pit_gpu}", flush=True)
sg = ds.sigma()              # host copy, 34 GB
ds.close()
torch.cuda.empty_cache()

# ---- oracle: the reference's sweep order (solver.py:241-265), W per set on the fly
sigma = np.eye(p)
tcpu = 0.0
for k, idx in enumerate(part.sets):
    comp = orc.complement(p, idx)
    ts = time.perf_counter()
    op = orc.BlockOp(a, idx, comp)
    tsetup = time.perf_counter() - ts
    ts = time.perf_counter()
    op.apply(sigma)
    tapply = time.perf_counter() - ts
    tcpu += tapply
    del op
    print(f"oracle set {k}: b={len(idx)} setup {tsetup:.1f}s apply {tapply:.1f}s", flush=True)
idx = part.sets[-1]
comp = orc.complement(p, idx)
ts = time.perf_counter()
err_ref, pit_ref, conv = orc.error_estimate(a, sigma, idx, comp)
test = time.perf_counter() - ts
tcpu += test
print(f"oracle estimate {test:.1f}s: err {err_ref:.12e}, power iterations {pit_ref} (converged {conv}); "
      f"oracle sweep (block updates + estimate) {tcpu:.1f}s", flush=True)

# ---- compare in row chunks
num = den = 0.0
sym = 0.0
for lo in range(0, p, 4096):
    d = sg[lo:lo + 4096] - sigma[lo:lo + 4096]
    num += float(np.einsum("ij,ij->", d, d))
    den += float(np.einsum("ij,ij->", sigma[lo:lo + 4096], sigma[lo:lo + 4096]))
    sym = max(sym, float(np.max(np.abs(sg[lo:lo + 4096, :4096] - sg[:4096, lo:lo + 4096].T))))
rel = (num / den) ** 0.5
print(f"c5 sweep 1: Sigma rel Frobenius GPU vs oracle {rel:.3e} (bar 1e-10); "
      f"err rel diff {abs(err_gpu - err_ref) / err_ref:.3e}; GPU Sigma max asymmetry (first 4096 cols) {sym:.1e}",
      flush=True)
assert rel < 1e-10, rel
