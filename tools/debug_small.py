import os, subprocess, sys
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import paper_2502_06377_b200 as pkg
from paper_2502_06377_b200 import _abi
L = _abi.lib()
tma, split, p = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
L.ibmi_tune(3, tma); L.ibmi_tune(1, split); L.ibmi_tune(2, split)
m = np.random.default_rng(0).standard_normal((p, p)); a = m.T @ m + p * np.eye(p)
part = pkg.contiguous_partition(p, 2)
sig = np.eye(p) + 0.01
pkg.block_update(a, sig, part.sets[0], pkg.complement(part, 0))
print("ok", tma, split, p, float(np.abs(sig).sum()))
'''
for args in [("0", "0", "64"), ("1", "1", "64"), ("1", "0", "64"), ("1", "1", "256"), ("1", "1", "512"), ("1", "1", "96"), ("1", "1", "200")]:
    r = subprocess.run([sys.executable, "-c", code, *args], capture_output=True, text=True, env=dict(os.environ, **({"IBMI_DEBUG_SYNC": "1"} if len(sys.argv) < 2 else {})))
    print(args, r.returncode, r.stdout.strip()[-200:], "\n   ", "\n    ".join(r.stderr.strip().splitlines()[-6:]))
