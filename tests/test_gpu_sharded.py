"""Sharded sweep through the CUDA backend (libibmi_b200.so) on the one GPU of
the test box: a 1-rank NCCL group, and 2 ranks sharing the GPU over gloo
(collectives staged through the host, so no kernel waits on another rank)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, golden

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, backend, case, out, exchange="nccl", operands="auto"):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group(backend, rank=rank, world_size=world)
    try:
        from paper_2502_06377_b200 import configs, contiguous_partition
        from paper_2502_06377_b200.distributed import ShardedSolver

        name, sweeps, panel = case
        if name == "c1":
            cfg = configs.get_config("c1")
            a, part, guess = configs.make_matrix("c1"), cfg.partition(), "jacobi"
        else:
            p, k, f = name
            m = np.random.default_rng(p).standard_normal((p, p))
            a, part, guess = m.T @ m + p * np.eye(p), contiguous_partition(p, k, f), "identity"
        ss = ShardedSolver(a, part, panel=panel, device=0, exchange=exchange, operands=operands)
        if operands == "sharded":
            assert ss.W is None and ss.A.shape[0] == ss.n_loc
        if os.environ.get("IBMI_TEST_LATE_RANK") == str(rank):
            import time

            time.sleep(1.5)          # this rank seeds (and zeroes) its panel long after the others
        ss.init_sigma(guess)
        errs = [ss.sweep()[0] for _ in range(sweeps)]
        sig = ss.gather_sigma()
        fr = ss.frobenius()
        ss.close()
        out.put((rank, errs, sig, fr))
    finally:
        dist.destroy_process_group()


def _run(world, backend, case, exchange="nccl", operands="auto"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, case, q, exchange, operands)) for r in range(world)]
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
    return res


@pytest.mark.parametrize("world,backend,exchange,operands", [
    (1, "nccl", "nccl", "replicated"), (2, "gloo", "nccl", "replicated"), (1, "nccl", "p2p", "replicated"),
    (2, "gloo", "p2p", "replicated"), (1, "nccl", "p2p", "sharded"), (2, "gloo", "p2p", "sharded"),
    (2, "gloo", "nccl", "sharded")])
def test_sharded_c1_matches_reference(world, backend, exchange, operands):
    g = golden("c1.npz")
    res = _run(world, backend, ("c1", int(g["iterations"][0]), 128), exchange, operands)
    for rank, errs, sig, fr in res:
        assert np.linalg.norm(sig - g["sigma"]) <= 1e-10 * np.linalg.norm(g["sigma"])
        ref = g["error_trace"]
        assert np.all(np.abs(np.array(errs) - ref) <= 1e-6 * ref + 1e-12)
        assert fr < 1e-9


@pytest.mark.parametrize("exchange,operands", [("nccl", "replicated"), ("p2p", "replicated"), ("p2p", "sharded"),
                                               ("nccl", "sharded")])
@pytest.mark.parametrize("case", [((1024, 4, 0.125), 6, 128), ((520, 3, 0.1), 5, 64)])
def test_sharded_two_ranks_match_oracle(case, exchange, operands):
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import contiguous_partition

    (p, k, f), sweeps, panel = case
    res = _run(2, "gloo", case, exchange, operands)
    m = np.random.default_rng(p).standard_normal((p, p))
    a = m.T @ m + p * np.eye(p)
    o = orc.solve(a, contiguous_partition(p, k, f).sets, tol=1e-300, max_iterations=sweeps)
    for rank, errs, sig, fr in res:
        assert np.linalg.norm(sig - o["result"]) <= 1e-10 * np.linalg.norm(o["result"])
        np.testing.assert_allclose(errs, o["error_trace"], rtol=1e-6, atol=1e-13)


def test_sharded_operands_three_ranks():
    """Operand-sharded set-up and sweeps on 3 ranks sharing the GPU (uneven panels)."""
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import contiguous_partition

    case = ((600, 4, 0.1), 4, 64)
    (p, k, f), sweeps, panel = case
    res = _run(3, "gloo", case, "p2p", "sharded")
    m = np.random.default_rng(p).standard_normal((p, p))
    a = m.T @ m + p * np.eye(p)
    o = orc.solve(a, contiguous_partition(p, k, f).sets, tol=1e-300, max_iterations=sweeps)
    for rank, errs, sig, fr in res:
        assert np.linalg.norm(sig - o["result"]) <= 1e-10 * np.linalg.norm(o["result"])
        np.testing.assert_allclose(errs, o["error_trace"], rtol=1e-6, atol=1e-13)
        assert abs(fr - orc.frobenius_residual(a, o["result"])) <= 1e-9 * max(1.0, fr)


def _bad_worker(rank, world, port, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_06377_b200 import NotPositiveDefinite, contiguous_partition
        from paper_2502_06377_b200.distributed import ShardedSolver

        p = 256
        m = np.random.default_rng(3).standard_normal((p, p))
        a = m.T @ m + p * np.eye(p)
        a[200, 200] = -1.0                      # set 1 (owner: rank 1) is not SPD, local pivot 200 - lo
        part = contiguous_partition(p, 2, 0.0)
        try:
            ShardedSolver(a, part, panel=64, device=0, exchange="nccl", operands="sharded")
            out.put((rank, None))
        except NotPositiveDefinite as e:
            out.put((rank, (e.index, e.set_index)))
    finally:
        dist.destroy_process_group()


def test_sharded_operands_not_spd_raises_on_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bad_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert sorted(res) == [(0, (72, 1)), (1, (72, 1))]


def test_sharded_p2p_late_rank_cannot_wipe_peer_stores(monkeypatch):
    """in the fused p2p exchange K1's epilogue stores −M into the OWNERS' panels.
    A rank that zeroes its panel late (init_sigma) must not wipe stores of a rank that is
    already sweeping: init_sigma ends with a barrier.  Rank 1 enters init_sigma 1.5 s late."""
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import contiguous_partition

    monkeypatch.setenv("IBMI_TEST_LATE_RANK", "1")
    case = ((520, 3, 0.1), 3, 64)
    (p, k, f), sweeps, panel = case
    res = _run(2, "gloo", case, "p2p", "sharded")
    m = np.random.default_rng(p).standard_normal((p, p))
    a = m.T @ m + p * np.eye(p)
    o = orc.solve(a, contiguous_partition(p, k, f).sets, tol=1e-300, max_iterations=sweeps)
    for rank, errs, sig, fr in res:
        assert np.linalg.norm(sig - o["result"]) <= 1e-10 * np.linalg.norm(o["result"])
        np.testing.assert_allclose(errs, o["error_trace"], rtol=1e-6, atol=1e-13)


def _solve_worker(rank, world, port, guess, out):
    import sys

    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2502_06377_b200 import IbmiConfig, contiguous_partition
        from paper_2502_06377_b200.distributed import solve_sharded

        p = 520
        m = np.random.default_rng(p).standard_normal((p, p))
        a = m.T @ m + 0.05 * p * np.eye(p)
        rep = solve_sharded(a, contiguous_partition(p, 4, 0.125),
                            IbmiConfig(tol=1e-10, initial_guess=guess, max_iterations=200, mc_samples=40, mc_seed=3),
                            panel=64, device=0)
        out.put((rank, rep.iterations, rep.converged, rep.error_trace, rep.result))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("guess", ["local", "mc", "takahashi"])
def test_solve_sharded_reference_guesses(guess):
    """solve_sharded with the reference's non-trivial initial guesses (solver.py:162-222):
    Σ₀[c₁,c₁] is formed by the single-GPU kernels on every rank and seeded panel by panel."""
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import contiguous_partition

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_solve_worker, args=(r, 2, port, guess, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = 520
    m = np.random.default_rng(p).standard_normal((p, p))
    a = m.T @ m + 0.05 * p * np.eye(p)
    o = orc.solve(a, contiguous_partition(p, 4, 0.125).sets, tol=1e-10, guess=guess, max_iterations=200,
                  mc_samples=40, mc_seed=3)
    for rank, iters, conv, errs, sig in res:
        assert conv and abs(iters - o["iterations"]) <= 1
        assert np.linalg.norm(sig - o["result"]) <= 1e-10 * np.linalg.norm(o["result"])


@pytest.mark.parametrize("exchange", ["p2p", "nccl"])
def test_sharded_four_ranks_overlapping_mid_size(exchange):
    """Four ranks sharing the GPU, p = 2048 in 128-row block-cyclic panels (four panels per rank),
    eight overlapping sets, operands sharded: W panel gathers, fused peer-store exchange through
    CUDA IPC between four processes, split Gram — against the oracle."""
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import contiguous_partition

    case = ((2048, 8, 0.125), 4, 128)
    (p, k, f), sweeps, panel = case
    res = _run(4, "gloo", case, exchange, "sharded")
    m = np.random.default_rng(p).standard_normal((p, p))
    a = m.T @ m + p * np.eye(p)
    o = orc.solve(a, contiguous_partition(p, k, f).sets, tol=1e-300, max_iterations=sweeps)
    assert len(res) == 4
    for rank, errs, sig, fr in res:
        assert np.linalg.norm(sig - o["result"]) <= 1e-10 * np.linalg.norm(o["result"])
        np.testing.assert_allclose(errs, o["error_trace"], rtol=1e-6, atol=1e-13)
        assert abs(fr - orc.frobenius_residual(a, o["result"])) <= 1e-9 * max(1.0, fr)
