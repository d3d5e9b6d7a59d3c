import os
import subprocess
import sys

code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import random_spd
import paper_2502_06377_b200 as pkg
from paper_2502_06377_b200 import _abi
from paper_2502_06377_b200.device import DeviceSolver
from oracle import ibmi_oracle as orc
L = _abi.lib()
tma, split, clus, p, k, f = [float(x) for x in sys.argv[1:7]]
p, k = int(p), int(k)
L.ibmi_tune(3, int(tma)); L.ibmi_tune(1, int(split)); L.ibmi_tune(2, int(split)); L.ibmi_tune(4, int(split)); L.ibmi_tune(5, int(clus))
a = random_spd(p, p + k)
part = pkg.contiguous_partition(p, k, f)
ds = DeviceSolver(a, partition=part)
ds.setup(); ds.init_sigma(0)
sig = np.eye(p)
ops = [orc.BlockOp(a, s, orc.complement(p, s)) for s in part.sets]
out = []
for sweep in range(2):
    for j in range(k):
        ds.block_update(j); ops[j].apply(sig)
        d = ds.sigma()
        out.append(f"{sweep}.{j}:{np.abs(d - sig).max():.1e}")
print("tma", int(tma), "split", int(split), "clus", int(clus), " ".join(out))
'''
for args in [("1", "0", "1"), ("0", "0", "1"), ("1", "1", "1"), ("0", "1", "1"), ("0", "1", "0")]:
    for shape in [("9", "4", "0.0"), ("600", "7", "0.0")]:
        r = subprocess.run([sys.executable, "-c", code, *args, *shape], capture_output=True, text=True)
        print(shape, r.stdout.strip()[-400:], r.stderr.strip()[-300:])
