"""Sharded sweep (paper_2502_06377_b200.distributed) on CPU with gloo.

world_size 2 and 3, block-cyclic panels of 8 rows, the torch CPU emulation of
the GEMM backend (tests/torch_backend.py).  Every rank must end with the
oracle's Σ (relative Frobenius ≤ 1e-12), error trace and ‖I − AΣ‖_F.
"""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, out):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from torch_backend import TorchCPUBackend

        from paper_2502_06377_b200 import contiguous_partition, red_black_partition
        from paper_2502_06377_b200.distributed import ShardedSolver

        p, k, f, sweeps, guess = case[:5]
        operands = case[5] if len(case) > 5 else "replicated"
        m = np.random.default_rng(p + k).standard_normal((p, p))
        a = m.T @ m + p * np.eye(p)
        part = red_black_partition(p) if k == 0 else contiguous_partition(p, k, f)
        ss = ShardedSolver(a, part, panel=8, backend=TorchCPUBackend(), operands=operands)
        assert ss.operands == operands
        if operands == "sharded":
            assert ss.W is None and ss.A.shape[0] == ss.n_loc      # nothing of order p² replicated
        ss.init_sigma(guess)
        errs = [ss.sweep()[0] for _ in range(sweeps)]
        sig = ss.gather_sigma()
        fr = ss.frobenius()
        out.put((rank, errs, sig, fr))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (w, c) for w in (2, 3) for c in [(96, 3, 0.1, 4, "identity"), (80, 2, 0.0, 3, "jacobi"),
                                     (64, 0, 0.0, 3, "identity"), (100, 4, 0.2, 3, "identity")]
] + [
    # operands sharded: A row panels, W column shards gathered per step, set-up split over the ranks
    (2, (96, 3, 0.1, 4, "identity", "sharded")), (2, (80, 2, 0.0, 3, "jacobi", "sharded")),
    (3, (100, 4, 0.2, 3, "identity", "sharded")), (4, (96, 3, 0.1, 4, "identity", "sharded")),
    (4, (64, 0, 0.0, 3, "identity", "sharded")), (5, (100, 5, 0.2, 2, "jacobi", "sharded")),
    (4, (96, 3, 0.1, 4, "identity")),
])
def test_sharded_matches_oracle(world, case):
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import contiguous_partition, red_black_partition

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    import queue
    import time as _time

    res, deadline = [], _time.time() + 240
    while len(res) < len(procs):
        try:
            res.append(q.get(timeout=2))
        except queue.Empty:
            dead = [pr.exitcode for pr in procs if pr.exitcode not in (None, 0)]
            if dead or _time.time() > deadline:
                for pr in procs:
                    pr.kill()
                raise AssertionError(f"worker failed (exit codes {[pr.exitcode for pr in procs]})")
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p, k, f, sweeps, guess = case[:5]
    m = np.random.default_rng(p + k).standard_normal((p, p))
    a = m.T @ m + p * np.eye(p)
    part = red_black_partition(p) if k == 0 else contiguous_partition(p, k, f)
    o = orc.solve(a, part.sets, tol=1e-300, max_iterations=sweeps, guess=guess)
    for rank, errs, sig, fr in res:
        assert np.linalg.norm(sig - o["result"]) <= 1e-12 * np.linalg.norm(o["result"]), rank
        np.testing.assert_allclose(errs, o["error_trace"], rtol=1e-6, atol=1e-14)
        assert abs(fr - orc.frobenius_residual(a, o["result"])) <= 1e-9 * max(1.0, fr)


def _solve_worker(rank, world, port, case, out):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from torch_backend import TorchCPUBackend

        from paper_2502_06377_b200 import IbmiConfig, contiguous_partition
        from paper_2502_06377_b200.distributed import solve_sharded

        p, k, f, tol, guess, stopping = case
        m = np.random.default_rng(p + k).standard_normal((p, p))
        a = m.T @ m + 0.05 * p * np.eye(p)
        part = contiguous_partition(p, k, f)
        s0 = None
        if guess not in ("identity", "jacobi"):       # CPU test: Σ₀[c₁,c₁] from the oracle's guess
            from oracle import ibmi_oracle as orc

            comp0 = orc.complement(p, part.sets[0])
            s0 = orc.initial_sigma(a, comp0, guess)[np.ix_(comp0, comp0)]
        rep = solve_sharded(a, part,
                            IbmiConfig(tol=tol, initial_guess=guess, stopping=stopping, max_iterations=300),
                            panel=8, backend=TorchCPUBackend(), sigma0_cc=s0)
        out.put((rank, rep.iterations, rep.converged, rep.error_trace, rep.result, rep.residual_trace))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [(72, 3, 0.1, 1e-10, "identity", "estimate"),
                                  (64, 2, 0.0, 1e-9, "jacobi", "frobenius"),
                                  (72, 3, 0.1, 1e-10, "local", "estimate")])
def test_solve_sharded_matches_oracle(case):
    """solve_sharded (the public N-rank solve) stops on the same sweep as the oracle's solve."""
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import contiguous_partition

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p, k, f, tol, guess, stopping = case
    m = np.random.default_rng(p + k).standard_normal((p, p))
    a = m.T @ m + 0.05 * p * np.eye(p)
    o = orc.solve(a, contiguous_partition(p, k, f).sets, tol=tol, guess=guess, stopping=stopping,
                  max_iterations=300)
    assert o["converged"]
    for rank, iters, conv, errs, sig, resid in res:
        assert conv and iters == o["iterations"], (rank, iters, o["iterations"])
        np.testing.assert_allclose(errs, o["error_trace"], rtol=1e-6, atol=1e-2 * tol)
        assert np.linalg.norm(sig - o["result"]) <= 1e-10 * np.linalg.norm(o["result"])
        if stopping == "frobenius":
            assert resid[-1] < tol and len(resid) == iters
