"""c4 through the FP64 floor on the GPU against the reference-generated fixture
(tests/golden/c4long.npz: the reference's own sweeps at tol 1e-8, 30 sweeps).

Prints, per sweep, the GPU error estimate next to the reference's, and at every
fixture checkpoint the sketch / row-sum / sample / ‖Σ‖_F distances and
‖I − AΣ‖_F.  Measurement behind the c4 tolerance decision and
the bounds asserted by tests/test_gpu_parity.py::test_c4_through_the_floor.

usage: python tools/c4_long_compare.py [moduli]     (0 = FP64 DMMA, default)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2502_06377_b200 import configs  # noqa: E402
from paper_2502_06377_b200.device import DeviceSolver  # noqa: E402

moduli = int(sys.argv[1]) if len(sys.argv) > 1 else 0
g = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "c4long.npz"))
cfg = configs.get_config("c4")
a = configs.make_matrix("c4")
r = np.random.default_rng(2025).standard_normal((cfg.p, g[f"snap{int(g['checkpoints'][0])}_sketch"].shape[1]))
ref = g["error_trace"]
cps = set(int(c) for c in g["checkpoints"])
with DeviceSolver(a, partition=cfg.partition()) as ds:
    if moduli:
        ds.set_emulation(moduli)
    ds.setup()
    ds.init_sigma(0)
    for it in range(1, len(ref) + 1):
        err, pit, _ = ds.sweep(1e-9, 5000)
        line = f"sweep {it:2d} gpu {err:.6e} ref {ref[it - 1]:.6e} rel {abs(err - ref[it - 1]) / ref[it - 1]:.2e} pit {pit}/{int(g['power_iters'][it - 1])}"
        if it in cps:
            s = ds.sigma()
            fro = float(g[f"snap{it}_fro"][0])
            sk = np.linalg.norm(s @ r - g[f"snap{it}_sketch"]) / np.linalg.norm(g[f"snap{it}_sketch"])
            sm = np.linalg.norm(s[g["sample_i"], g["sample_j"]] - g[f"snap{it}_sample"]) / np.linalg.norm(g[f"snap{it}_sample"])
            rs = np.linalg.norm(s.sum(axis=1) - g[f"snap{it}_rowsum"]) / (fro * np.sqrt(cfg.p))
            fr = ds.frobenius()
            line += (f" | sketch {sk:.2e} sample {sm:.2e} rowsum/(fro sqrt p) {rs:.2e} dfro {abs(np.linalg.norm(s) - fro) / fro:.2e}"
                     f" frob gpu {fr:.4e} ref {float(g[f'snap{it}_frobenius'][0]):.4e}")
        print(line, flush=True)
