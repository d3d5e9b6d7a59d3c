"""bench.py's output contract: stdout is exactly one JSON line with the keys the
driver reads.  The reference arm runs on CPU (the oracle port at c1); our arm
needs the GPU."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, res.stdout[-3000:]
    return json.loads(lines[0])


def test_reference_arm_line_on_cpu():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"], timeout=600)
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["e2e"]["d2h_bytes_per_step"] == 0
    # each step is one whole sweep, timed: the claimed time fits the sweeps reported
    assert d["steps"] == 2 and len(d["sweep_seconds"]) == 2
    assert abs(d["ms_per_step"] - 1e3 * sum(d["sweep_seconds"]) / 2) < 1e-6 * d["ms_per_step"]
    assert abs(d["value"] - 2 / sum(d["sweep_seconds"])) < 1e-9 * d["value"]
    # the same error trace as the reference's first two c1 sweeps (golden fixture)
    from conftest import golden

    # (bit-equal with the fixture's BLAS thread count; other thread counts move the last bits)
    np.testing.assert_allclose(d["error_trace"], golden("c1.npz")["error_trace"][:2], rtol=1e-12, atol=0)
    assert "cpu_model" in cb and "blas" in cb
    assert set(d["config"]) == {"workload", "p", "sets", "overlap", "set_sizes", "l2"}


def test_reference_arm_budget_caps_sweeps():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "50", "--warmup", "0", "--ref-budget-s", "0"],
             timeout=600)
    assert d["steps"] == 1 and len(d["sweep_seconds"]) == 1 and "capped" in d["cpu_baseline"]["sample"]


def test_gpus_flag_never_measures_on_fewer_gpus():
    """--gpus N outside torchrun either launches N ranks or exits non-zero; a
    WORLD_SIZE that disagrees with --gpus is an error."""
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "64", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 3 and res.stdout.strip() == "", (res.returncode, res.stdout[-500:])
    assert "needs 64 GPUs" in res.stderr
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--steps", "1"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert res.returncode == 2 and res.stdout.strip() == ""


@pytest.mark.gpu
def test_our_arm_line_on_gpu():
    d = _run(["--config", "c1", "--steps", "3", "--warmup", "3", "--no-alt", "--no-cpu-baseline"], timeout=900)
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "f64" and d["config"]["workload"].startswith("c1")
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] <= 1.05
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
@pytest.mark.parametrize("operands", ["replicated", "sharded"])
def test_sharded_driver_line_on_gpu(operands):
    """The N-rank driver of bench.py at world size 1 (`--sharded`): same contract keys, plus the
    `sharded` block (operand mode, exchange, this rank's NVLink bytes per sweep) and an e2e
    through solve_sharded."""
    d = _run(["--config", "c1", "--steps", "3", "--warmup", "3", "--no-alt", "--no-cpu-baseline", "--sharded",
              "--operands", operands], timeout=900)
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    sh = d["sharded"]
    assert sh["operands"] == operands and sh["exchange_mode"] in ("p2p", "nccl")
    assert sh["comm_bytes_per_sweep_this_rank"]["gemm_flops"] > 0
    assert sh["comm_bytes_per_sweep_this_rank"]["exchange_out"] == 0      # one rank: nothing crosses NVLink
    assert d["time_to_tol"]["sweeps"] == 107
    assert d["e2e"]["value"] > 0
