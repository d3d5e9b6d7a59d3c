"""Freeze the reference algorithm's first c5 sweep (p = 65536) as a fixture.

Runs on the GPU box (A is generated on the GPU by configs.make_matrix_c5_device
and needs ~140 GB of host RAM for the CPU side).  The oracle (oracle/ibmi_oracle.py,
the reference algorithm on NumPy/OpenBLAS, bit-identical to the reference on the
pinned cases) runs the first sweep in solve()'s order (solver.py:241-265) from
Σ₀ = I; W_k is formed per set on the fly (same arithmetic, 39 GB less RAM).

Writes gpurun_out/c5.npz + c5.json (copy them to tests/golden/): the error
estimate and its power-iteration count, the sketch Σ·R (R = seeded Gaussian
65536 × 4, make_golden.sketch_matrix), row sums, ‖Σ‖_F, 4096 sampled entries,
and a checksum of A so the GPU test knows it regenerated the same matrix.
This is test infrastructure: only tests/ read the fixture.
"""
import json
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", str(os.cpu_count() or 1))
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import ibmi_oracle as orc  # noqa: E402
from paper_2502_06377_b200 import configs  # noqa: E402

SKETCH_SEED, SKETCH_COLS, SAMPLE_SEED, N_SAMPLES = 2025, 4, 12345, 4096   # as tests/golden/make_golden.py

cfg = configs.get_config("c5")
part = cfg.partition()
p = cfg.p
t0 = time.perf_counter()
a_dev = configs.make_matrix_c5_device(0)
a = a_dev.cpu().numpy()
del a_dev
torch.cuda.empty_cache()
checksum = [float(a.sum()), float(np.linalg.norm(a)), float(a[0, 0]), float(a[-1, -1]), float(a[123, 45678])]
print(f"A generated on the GPU, copied to host in {time.perf_counter() - t0:.1f}s; checksum {checksum}", flush=True)

sigma = np.eye(p)
tsweep = 0.0
for k, idx in enumerate(part.sets):
    comp = orc.complement(p, idx)
    op = orc.BlockOp(a, idx, comp)
    ts = time.perf_counter()
    op.apply(sigma)
    tsweep += time.perf_counter() - ts
    del op
    print(f"oracle set {k}: b={len(idx)} done ({tsweep:.0f}s of block updates)", flush=True)
idx = part.sets[-1]
comp = orc.complement(p, idx)
ts = time.perf_counter()
err, pit, conv = orc.error_estimate(a, sigma, idx, comp)
tsweep += time.perf_counter() - ts
print(f"oracle estimate: err {err:.15e} power iterations {pit} (converged {conv}); sweep {tsweep:.0f}s", flush=True)

r = np.random.default_rng(SKETCH_SEED).standard_normal((p, SKETCH_COLS))
rng = np.random.default_rng(SAMPLE_SEED)
si, sj = rng.integers(0, p, N_SAMPLES), rng.integers(0, p, N_SAMPLES)
sketch = np.zeros((p, SKETCH_COLS))
rowsum = np.zeros(p)
fro2 = 0.0
for lo in range(0, p, 4096):
    blk = sigma[lo:lo + 4096]
    sketch[lo:lo + 4096] = blk @ r
    rowsum[lo:lo + 4096] = blk.sum(axis=1)
    fro2 += float(np.einsum("ij,ij->", blk, blk))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
np.savez_compressed(os.path.join(ROOT, "gpurun_out", "c5.npz"), sweep1_sketch=sketch, sweep1_rowsum=rowsum,
                    sweep1_fro=np.array([fro2 ** 0.5]), sweep1_sample=sigma[si, sj], sample_i=si, sample_j=sj,
                    error_trace=np.array([err]), power_iters=np.array([pit]), a_checksum=np.array(checksum))
meta = {"config": "c5", "p": p, "k": part.k, "sweeps": 1, "error_trace": [err], "power_iters": [int(pit)],
        "oracle_sweep_seconds": tsweep, "host_threads": os.cpu_count(),
        "openblas_threads": os.environ["OPENBLAS_NUM_THREADS"], "numpy": np.__version__, "torch": torch.__version__,
        "sketch_cols": SKETCH_COLS, "sketch_seed": SKETCH_SEED, "a_checksum": checksum,
        "generator": "configs.make_matrix_c5_device(0): torch Philox normals on the GPU, B B^T / p + 0.5 I"}
with open(os.path.join(ROOT, "gpurun_out", "c5.json"), "w") as fh:
    json.dump(meta, fh, indent=1)
print("c5 fixture written", meta, flush=True)
