"""The library's device block cache (ibmi_release_cached_memory / ibmi_cached_bytes):
a second solve of the same shape reuses the first one's blocks and returns the
identical Σ; blocks handed out dirty (IBMI_MEM_POISON=1, every block filled with
NaN bytes) still give the reference's answer, so no kernel reads memory it did
not write first."""

from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, random_spd

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need CUDA (run with -m 'not gpu' on CPU hosts)")
    import paper_2502_06377_b200 as pkg

    pkg.load_library()


def test_repeat_solve_reuses_blocks_and_is_identical():
    import paper_2502_06377_b200 as pkg

    p = 640
    a = random_spd(p, seed=11)
    part = pkg.contiguous_partition(p, 4, 0.125)
    cfg = pkg.IbmiConfig(tol=1e-11)
    pkg.release_cached_memory()
    assert pkg.cached_bytes() == 0
    r1 = pkg.solve(a, part, cfg)
    held = pkg.cached_bytes(0)
    assert held >= 2 * p * p * 8            # at least A and Σ came back to the cache
    r2 = pkg.solve(a, part, cfg)
    assert pkg.cached_bytes(0) <= held      # served from the cache, nothing new reserved
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.result, r2.result)
    assert r1.error_trace == r2.error_trace
    pkg.release_cached_memory(0)
    assert pkg.cached_bytes(0) == 0


_POISON_SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import paper_2502_06377_b200 as pkg
from conftest import random_spd
from oracle import ibmi_oracle as orc

cases = [(384, 3, 0.125, "identity"), (512, 2, 0.0, "jacobi"), (448, 4, 0.25, "local")]
for gemm in ("dmma", "ozaki"):
    for p, k, f, guess in cases:
        a = random_spd(p, seed=p + k)
        part = pkg.contiguous_partition(p, k, f)
        for _ in range(2):                   # the second solve runs on recycled (poisoned) blocks
            rep = pkg.solve(a, part, pkg.IbmiConfig(tol=1e-10, initial_guess=guess, gemm=gemm))
        ref = orc.solve(a, part.sets, tol=1e-10, guess=guess)
        rel = np.linalg.norm(rep.result - ref["result"]) / np.linalg.norm(ref["result"])
        assert np.isfinite(rep.result).all(), (gemm, p, k, guess)
        assert rel < 1e-10 and abs(rep.iterations - ref["iterations"]) <= 1, (gemm, p, k, guess, rel)
rb = pkg.red_black_partition(512)
a = random_spd(512, seed=5)
rep = pkg.solve(a, rb, pkg.IbmiConfig(tol=1e-10))
ref = orc.solve(a, rb.sets, tol=1e-10)
assert np.linalg.norm(rep.result - ref["result"]) / np.linalg.norm(ref["result"]) < 1e-10
print("poison ok")
"""


def test_poisoned_blocks_give_reference_results():
    env = dict(os.environ, IBMI_MEM_POISON="1")
    script = _POISON_SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"))
    res = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0 and "poison ok" in res.stdout, res.stdout[-3000:] + res.stderr[-3000:]
