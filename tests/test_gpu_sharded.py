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


def _worker(rank, world, port, backend, case, out, exchange="nccl"):
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
        ss = ShardedSolver(a, part, panel=panel, device=0, exchange=exchange)
        ss.init_sigma(guess)
        errs = [ss.sweep()[0] for _ in range(sweeps)]
        sig = ss.gather_sigma()
        fr = ss.frobenius()
        ss.close()
        out.put((rank, errs, sig, fr))
    finally:
        dist.destroy_process_group()


def _run(world, backend, case, exchange="nccl"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, backend, case, q, exchange)) for r in range(world)]
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


@pytest.mark.parametrize("world,backend,exchange", [(1, "nccl", "nccl"), (2, "gloo", "nccl"), (1, "nccl", "p2p"),
                                                     (2, "gloo", "p2p")])
def test_sharded_c1_matches_reference(world, backend, exchange):
    g = golden("c1.npz")
    res = _run(world, backend, ("c1", int(g["iterations"][0]), 128), exchange)
    for rank, errs, sig, fr in res:
        assert np.linalg.norm(sig - g["sigma"]) <= 1e-10 * np.linalg.norm(g["sigma"])
        ref = g["error_trace"]
        assert np.all(np.abs(np.array(errs) - ref) <= 1e-6 * ref + 1e-12)
        assert fr < 1e-9


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
@pytest.mark.parametrize("case", [((1024, 4, 0.125), 6, 128), ((520, 3, 0.1), 5, 64)])
def test_sharded_two_ranks_match_oracle(case, exchange):
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import contiguous_partition

    (p, k, f), sweeps, panel = case
    res = _run(2, "gloo", case, exchange)
    m = np.random.default_rng(p).standard_normal((p, p))
    a = m.T @ m + p * np.eye(p)
    o = orc.solve(a, contiguous_partition(p, k, f).sets, tol=1e-300, max_iterations=sweeps)
    for rank, errs, sig, fr in res:
        assert np.linalg.norm(sig - o["result"]) <= 1e-10 * np.linalg.norm(o["result"])
        np.testing.assert_allclose(errs, o["error_trace"], rtol=1e-6, atol=1e-13)
