"""Build libibmi_b200.so in-tree with nvcc for sm_100a (no torch JIT cache).

``python -m paper_2502_06377_b200.build`` or ``__graft_entry__.build()``.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libibmi_b200.so")
SOURCES = [os.path.join(HERE, "csrc", "ibmi_b200.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in ("common.cuh", "gemm_nt.cuh", "gemm_tma.cuh", "small_kernels.cuh", "small_sweep.cuh", "igemm_tc.cuh", "ozaki.cuh")] + [
    os.path.join(ROOT, "include", "ibmi_b200.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-pthread", "-shared", "--expt-relaxed-constexpr", "-Xptxas", "-v"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or stale():
        cmd = [NVCC, *FLAGS, "-o", LIB, *SOURCES, "-lcudart"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed building libibmi_b200.so")
        with open(os.path.join(HERE, "csrc", "ptxas.log"), "w") as fh:
            fh.write(res.stderr)
        if verbose:
            sys.stderr.write(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
