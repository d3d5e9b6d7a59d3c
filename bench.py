"""IBMI sweep benchmark (BASELINE metric: sweeps/s + FP64 TFLOP/s at p=16384).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One "step" is one IBMI sweep of the BASELINE config (default c4: p=16384,
Matérn-3/2 on x-sorted points, contiguous_partition(16384, 8, 0.125)): eight
block updates and the reference's error estimate on the last set
(solver.py:257-265).  Inputs (A, 2.15 GB; Σ, 2.15 GB) exceed the 126 MB L2,
so no explicit flush is needed between sweeps.

Our arm prints ONE JSON line on rank 0 with the device-timed sweeps/s
(``value``), the end-to-end number through the public ``solve`` API with host
buffers (``e2e``), the panel-GEMM roofline against the FP64 DMMA peak measured
on this box, the CPU oracle timed on a bounded sample (``cpu_baseline``) and
the SM clocks sampled during the timed region.

``--impl reference`` times the CPU oracle port (oracle/ibmi_oracle.py, the
reference algorithm on NumPy/SciPy OpenBLAS, all host threads) on the same
config: each timed step is one FULL sweep in the reference's order (K block
updates + the error estimate, solver.py:257-266), from the reference's Σ₀;
warm-up steps are single block updates (then Σ is reset), and the timed sweeps
stop early, with ``steps`` reporting the sweeps actually run, if the next one
would pass ``--ref-budget-s``.

``--gpus N`` without torchrun re-launches this script under
``torch.distributed.run`` with N ranks when the node has N GPUs, and exits
non-zero when it has fewer: a multi-GPU line is never measured on one GPU.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

_JSON_OUT = sys.stdout   # replaced by a private dup of fd 1 when run as a script

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="use the sharded driver even at N=1 (diagnostic)")
    ap.add_argument("--no-ttt", action="store_true", help="skip the time-to-tolerance run")
    ap.add_argument("--exchange", default="auto", choices=["auto", "nccl", "p2p"])
    ap.add_argument("--operands", default="auto", choices=["auto", "replicated", "sharded"],
                    help="sharded driver: A and W replicated, or A row panels + W column shards gathered per step "
                         "(auto: sharded when N > 1)")
    ap.add_argument("--gemm", default="dmma", choices=["dmma", "ozaki"],
                    help="headline GEMM path: FP64 DMMA (default) or Ozaki-II INT8 emulation")
    ap.add_argument("--moduli", type=int, default=16, help="Ozaki-II moduli (8..20)")
    ap.add_argument("--no-alt", action="store_true", help="skip measuring the other GEMM path")
    ap.add_argument("--ref-budget-s", type=float, default=1500.0,
                    help="reference arm: stop the timed sweeps before this many seconds")
    return ap.parse_args()


def bench_config(cfg, part) -> dict:
    """The workload description both arms print (so the driver sees the same config)."""
    sizes = [len(s) for s in part.sets]
    mat = cfg.p * cfg.p * 8
    l2 = ("inputs (A, Sigma: %.2f GB each) exceed the 126 MB L2; no flush" % (mat / 1e9) if mat > 126e6 else
          "inputs (A, Sigma: %.0f MB each) fit in L2; not flushed (every sweep rewrites all of Sigma)" % (mat / 1e6))
    return {"workload": f"{cfg.name}: {cfg.description}", "p": cfg.p, "sets": part.k, "overlap": cfg.overlap,
            "set_sizes": sorted(set(sizes)), "l2": l2}


def host_info() -> dict:
    """CPU model and the BLAS/LAPACK builds NumPy and SciPy run on."""
    import platform

    import scipy
    import scipy.linalg  # noqa: F401  (loads SciPy's OpenBLAS)

    model = platform.processor()
    try:
        with open("/proc/cpuinfo") as fh:
            model = next((ln.split(":", 1)[1].strip() for ln in fh if ln.startswith("model name")), model)
    except OSError:
        pass
    blas = []
    try:
        from threadpoolctl import threadpool_info

        for d in threadpool_info():
            blas.append({"api": d.get("internal_api"), "version": d.get("version"),
                         "threads": d.get("num_threads"), "arch": d.get("architecture"),
                         "lib": os.path.basename(d.get("filepath") or "")})
    except Exception as exc:  # noqa: BLE001 - informational only
        blas.append({"error": repr(exc)})
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "numpy": np.__version__, "scipy": scipy.__version__,
            "blas": blas}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


class ClockSampler:
    """SM clocks + throttle reasons sampled while running: NVML every 20 ms
    (so even a sub-second timed region gets samples), else nvidia-smi -lms 200."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits (nvml.h)
    BITS = {"sw_power_cap": 0x4, "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40}

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []          # (sm_mhz, max_mhz, reasons)
        self._stop = threading.Event()
        self.t = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self._physical_index())
            self._sample_nvml()
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return self
        except Exception:           # noqa: BLE001 - no NVML: nvidia-smi
            self._nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self._physical_index()), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _physical_index(self) -> int:
        vis = os.environ.get("CUDA_VISIBLE_DEVICES")
        if vis:
            try:
                return int(vis.split(",")[self.index])
            except (ValueError, IndexError):
                pass
        return self.index

    def _sample_nvml(self):
        nv = self._nv
        sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
        try:
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:           # noqa: BLE001 - older binding name
            bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        self.samples.append((float(sm), float(mx), {n for n, b in self.BITS.items() if bits & b}))

    def _nvml_loop(self):
        while not self._stop.wait(0.02):
            try:
                self._sample_nvml()
            except Exception:       # noqa: BLE001
                return

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self._stop.set()
        if self._nv is not None:
            try:
                self._sample_nvml()
            except Exception:       # noqa: BLE001
                pass
            if self.t:
                self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for a, b, r in self.samples:
            sm.append(a)
            mx.append(b)
            reasons |= r
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml 20 ms" if self.samples else "nvidia-smi 200 ms"}


def cpu_sample(cfg, a, n_blocks=1):
    """Time the CPU oracle (reference algorithm, NumPy/SciPy OpenBLAS) on a
    bounded sample and extrapolate to sweeps/s by the per-set FLOP model."""
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import configs

    part = cfg.partition()
    p = cfg.p
    k_mid = part.k // 2
    idx = part.sets[k_mid]
    comp = orc.complement(p, idx)
    t0 = time.perf_counter()
    op = orc.BlockOp(a, idx, comp)
    t_setup = time.perf_counter() - t0
    sigma = np.eye(p)
    times = []
    for _ in range(n_blocks):
        t0 = time.perf_counter()
        op.apply(sigma)
        times.append(time.perf_counter() - t0)
    lidx = part.sets[-1]
    lcomp = orc.complement(p, lidx)
    t0 = time.perf_counter()
    orc.error_estimate(a, sigma, lidx, lcomp)
    t_err = time.perf_counter() - t0
    b, c = len(idx), p - len(idx)
    per_flop = min(times) / (2.0 * b * c * c + 2.0 * b * b * c)
    sizes = [len(s) for s in part.sets]
    t_blocks = sum(per_flop * (2.0 * s * (p - s) ** 2 + 2.0 * s * s * (p - s)) for s in sizes)
    t_sweep = t_blocks + t_err
    return {"sweep_s": t_sweep, "block_s": min(times), "err_s": t_err, "setup_one_set_s": t_setup,
            "sample": f"{n_blocks} block update(s) of set {k_mid} (b={b}) + 1 error estimate on set {part.k - 1}, "
                      f"extrapolated to all {part.k} sets by the per-set FLOP model",
            "flops_per_sweep": configs.sweep_flops(cfg)}


def run_reference(args):
    """The reference's CPU path (oracle port, bit-identical to the reference on
    the pinned cases) timed in whole sweeps: solver.py:257-266 order, K block
    updates then the error estimate on the last set, from the reference Σ₀."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import ibmi_oracle as orc
    from paper_2502_06377_b200 import configs

    cfg = configs.get_config(args.config)
    if args.config == "c5":
        print(json.dumps({"impl": "reference", "unavailable": "c5's reference sweep needs ~140 GB of host RAM and "
                          "~21 min per sweep; run tools/c5_oracle_check.py instead"}), file=_JSON_OUT, flush=True)
        return
    a = configs.make_matrix(args.config)
    part = cfg.partition()
    p = cfg.p
    comps = [orc.complement(p, s) for s in part.sets]
    t0 = time.perf_counter()
    ops = [orc.BlockOp(a, part.sets[k], comps[k]) for k in range(part.k)]
    setup_s = time.perf_counter() - t0

    def sigma0():
        sig = np.eye(p)
        if cfg.guess == "jacobi":
            c0 = comps[0]
            sig[c0, c0] = 1.0 / np.diag(a)[c0]
        return sig

    sigma = sigma0()
    t_warm = time.perf_counter()
    for step in range(args.warmup):          # warm-up: single block updates (BLAS threads, page-in)
        ops[step % part.k].apply(sigma)
    warm_s = time.perf_counter() - t_warm
    sigma = sigma0()
    sweep_t, errs, pits = [], [], []
    t_start = time.perf_counter()
    for _ in range(args.steps):
        t1 = time.perf_counter()
        for op in ops:
            op.apply(sigma)
        e, it, _ = orc.error_estimate(a, sigma, part.sets[-1], comps[-1])
        sweep_t.append(time.perf_counter() - t1)
        errs.append(e)
        pits.append(it)
        elapsed = time.perf_counter() - t_start
        if elapsed + max(sweep_t) > args.ref_budget_s and len(sweep_t) < args.steps:
            break
    n = len(sweep_t)
    total = sum(sweep_t)
    value = n / total
    info = host_info()
    sample = (f"{n} full sweeps timed (each: {part.k} block updates + the error estimate on set {part.k - 1}, "
              f"solver.py:257-266 order, from the reference Sigma0)"
              + (f"; capped at {n} of {args.steps} by --ref-budget-s {args.ref_budget_s:.0f}" if n < args.steps else "")
              + f"; {args.warmup} warm-up steps = single block updates ({warm_s:.1f} s), then Sigma reset")
    line = {
        "impl": "reference",
        "metric": "IBMI sweeps/s (FP64) at p=16384" if args.config == "c4" else f"IBMI sweeps/s ({args.config})",
        "value": value, "unit": "sweeps/s", "n_gpus": world if world > 1 else args.gpus, "steps": n,
        "warmup": args.warmup, "ms_per_step": total / n * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(cfg, part),
        "tflops": configs.sweep_flops(cfg) * value / 1e12,
        "sweep_seconds": sweep_t, "error_trace": errs, "power_iterations": pits, "setup_s": setup_s,
        "cpu_baseline": {"value": value, "unit": "sweeps/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": sample, **info},
        "e2e": {"value": value, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), file=_JSON_OUT, flush=True)


def panel_traffic(name: str) -> dict:
    """`roofline.traffic` of the panel GEMM: ncu DRAM bytes per launch, measured per
    config on the committed code (tools/panel_traffic.py -> profiles/*_panel_traffic.json);
    null when no capture of this config is committed."""
    best = None
    prof = os.path.join(ROOT, "profiles")
    for fn in sorted(os.listdir(prof)) if os.path.isdir(prof) else []:
        if fn.endswith("_panel_traffic.json"):
            try:
                with open(os.path.join(prof, fn)) as fh:
                    d = json.load(fh).get(name)
            except (OSError, ValueError):
                d = None
            if d:
                best = (fn, d)           # the latest round's file wins
    if best is None:
        return {"traffic": None, "traffic_note": "no ncu DRAM capture of this config committed"}
    fn, d = best
    return {"traffic": d["bytes_per_launch"],
            "traffic_algorithmic": d["algorithmic_bytes_per_launch"],
            "traffic_note": f"profiles/{fn}: {d['how']}; read {d['read_per_launch']:.3e} + written "
                            f"{d['write_per_launch']:.3e} B per launch against an algorithmic "
                            f"{d['algorithmic_bytes_per_launch']:.3e} (W + Sigma_cc read once, M written twice); "
                            "operands exceed L2 at c3/c4, so resident CTAs re-stream them while the DMMA pipe is the bound"}


def executed_flops(cfg):
    """FLOPs the kernels actually execute per sweep: K2 and the Gram product
    compute only the lower triangle of a symmetric result."""
    part = cfg.partition()
    p = cfg.p
    tot = 0.0
    for s in part.sets:
        b = len(s)
        c = p - b
        tot += 2.0 * b * c * c + b * b * c
    b = len(part.sets[-1])
    c = p - b
    return tot + 2.0 * b * p * c + b * b * c


INT8_PEAK_TOPS = 4500.0   # B200 dense INT8 tensor peak (nominal, B200_PROFILING.md: fp8/int8 4.5 P dense)


def probe_int8_peak(n: int = 8192, reps: int = 10):
    """Measured INT8 tensor throughput on this box: cuBLASLt int8 GEMM
    (torch._int_mm, n^3, best of `reps`, CUDA events) — the denominator of
    the emulated path's roofline (MEASURED_PEAKS.json has no INT8 entry)."""
    import torch

    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t()
    for _ in range(3):
        torch._int_mm(a, b)
    best = float("inf")
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch._int_mm(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def measure_single(solver, cfg, args, stream, guess, mode, moduli, setup_s0):
    """Timed sweeps, per-kernel-class breakdown and time to tolerance of one
    GEMM mode ("dmma" or "ozaki") on a prepared single-GPU DeviceSolver."""
    import torch
    from paper_2502_06377_b200 import _abi as abi_mod

    L = abi_mod.lib()
    t0 = time.perf_counter()
    solver.set_emulation(moduli if mode == "ozaki" else 0)
    solver.init_sigma(1 if guess == "jacobi" else 0)
    for _ in range(args.warmup):          # first sweep also builds the residue-plane caches
        solver.sweep(1e-9, 5000)
    torch.cuda.synchronize()
    errs = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = L.ibmi_launch_count()
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            errs.append(solver.sweep(1e-9, 5000))
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    launches = L.ibmi_launch_count() - launches0
    sigma = solver.sigma(on_device=True).clone() if cfg.p <= 32768 else None   # c5: Σ alone is 34 GB
    # per-kernel-class device times (CUDA events on the same stream), best of 2
    if mode == "ozaki":
        abi_mod.check(L.ibmi_tune(9, 1))
    timed = [solver.sweep_timed(1e-9, 5000)[3] for _ in range(2)]
    kt = {k: min(t[k] for t in timed) for k in timed[0]}
    igemm = None
    if mode == "ozaki":
        import ctypes as C

        tms, tops, nl = C.c_double(), C.c_double(), C.c_int()
        abi_mod.check(L.ibmi_emulation_timing(C.byref(tms), C.byref(tops), C.byref(nl)))
        abi_mod.check(L.ibmi_tune(9, 0))
        igemm = {"ms": tms.value / 2, "int8_ops": tops.value / 2, "launches": nl.value // 2}
    ttt = None
    if not args.no_ttt:
        solver.init_sigma(1 if guess == "jacobi" else 0)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        n_to_tol = 0
        for n_to_tol in range(1, cfg.max_iterations + 1):
            e, _, _ = solver.sweep(1e-9, 5000)
            # exact skip: ‖I − AΣ‖_F ≥ err, so the residual is needed only once err < tol
            fr = solver.frobenius() if cfg.stopping == "frobenius" and e < 1.01 * cfg.tol else None
            if cfg.stopping == "frobenius" and fr is None:
                continue
            if (fr < cfg.tol) if fr is not None else (e <= cfg.tol):
                break
        torch.cuda.synchronize()
        ttt = {"seconds": setup_s0 + time.perf_counter() - t1, "sweeps": n_to_tol, "tol": cfg.tol,
               "stopping": cfg.stopping, "setup_s": setup_s0}
    return {"ms": ms, "sweeps_s": args.steps / (ms / 1e3), "errs": errs, "launches": launches, "kt": kt,
            "igemm": igemm, "ttt": ttt, "sigma": sigma, "clocks": clk.summary(),
            "switch_s": time.perf_counter() - t0}


def max_over_ranks(x: float, dev: int) -> float:
    import torch

    if not torch.distributed.is_initialized() or torch.distributed.get_world_size() == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{dev}")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    import paper_2502_06377_b200 as pkg
    from paper_2502_06377_b200 import configs
    from paper_2502_06377_b200.device import DeviceSolver, probe_fp64_peak

    cfg = configs.get_config(args.config)
    part = cfg.partition()
    p = cfg.p
    a_host = configs.make_matrix(args.config) if args.config != "c5" else None
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    if a_host is not None:
        a_dev = torch.as_tensor(a_host, device=f"cuda:{dev}")
    else:
        a_dev = configs.make_matrix_c5_device(0, device=f"cuda:{dev}")
    torch.cuda.synchronize()
    peak = probe_fp64_peak(dev)
    int8_peak = None
    if args.gemm == "ozaki" or not args.no_alt:
        try:
            int8_peak = probe_int8_peak()
        except Exception:           # torch without int8 cuBLASLt: fall back to the nominal figure
            int8_peak = None
    flops = configs.sweep_flops(cfg)
    sizes = [len(s) for s in part.sets]
    guess = "jacobi" if cfg.guess == "jacobi" else "identity"

    if args.sharded and world == 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device(f"cuda:{dev}"))
    if world == 1 and not args.sharded:
        # untimed warm-up context: first-use costs of a fresh process (lazy module loading, cold
        # cudaMalloc of GB-sized blocks — 25-500 ms, erratic) are not the solver's set-up time
        if cfg.p <= 32768:
            with DeviceSolver(a_dev, partition=part, device=dev, stream=stream.cuda_stream) as warm:
                warm.setup()
                warm.init_sigma(1 if guess == "jacobi" else 0)
                warm.sweep(1e-9, 5000)
            torch.cuda.synchronize()
        solver = DeviceSolver(a_dev, partition=part, device=dev, stream=stream.cuda_stream)
        del a_dev
        t0 = time.perf_counter()
        solver.set_emulation(args.moduli if args.gemm == "ozaki" else 0)
        solver.setup()
        solver.init_sigma(1 if guess == "jacobi" else 0)
        torch.cuda.synchronize()
        setup_s = time.perf_counter() - t0
        head = measure_single(solver, cfg, args, stream, guess, args.gemm, args.moduli, setup_s)
        alt = None
        if not args.no_alt:
            alt_mode = "ozaki" if args.gemm == "dmma" else "dmma"
            alt = measure_single(solver, cfg, args, stream, guess, alt_mode, args.moduli, setup_s)
            alt["sigma_rel_fro_vs_headline"] = (
                float(torch.linalg.norm(alt["sigma"] - head["sigma"]) / torch.linalg.norm(head["sigma"]))
                if head["sigma"] is not None else None)
            alt["mode"] = alt_mode
            del alt["sigma"]
        del head["sigma"]
        solver.close()
        torch.cuda.empty_cache()
        ms, errs, launches, kt, ttt = head["ms"], head["errs"], head["launches"], head["kt"], head["ttt"]
        sweeps_s = head["sweeps_s"]
        ms_step = ms / args.steps
        consistent = None
        clocks = head["clocks"]
        sharded_info = None
    else:
        from paper_2502_06377_b200.distributed import ShardedSolver

        t0 = time.perf_counter()
        solver = ShardedSolver(a_host if a_host is not None else a_dev, part, device=dev, exchange=args.exchange,
                               operands=args.operands)
        solver.init_sigma(guess)
        torch.cuda.synchronize()
        setup_s = time.perf_counter() - t0
        del a_dev
        sweep = lambda: solver.sweep(1e-9, 5000)          # noqa: E731
        for _ in range(args.warmup):
            sweep()
        errs = []
        torch.distributed.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        from paper_2502_06377_b200 import _abi as abi_mod

        launches0 = abi_mod.lib().ibmi_launch_count()
        with ClockSampler(dev) as clk:
            e0.record(stream)
            for _ in range(args.steps):
                errs.append(sweep())
            e1.record(stream)
            torch.cuda.synchronize()
        torch.distributed.barrier()
        ms = e0.elapsed_time(e1)
        launches = abi_mod.lib().ibmi_launch_count() - launches0
        if world > 1:
            t = torch.tensor([ms], device=f"cuda:{dev}")
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        ms_step = ms / args.steps
        sweeps_s = args.steps / (ms / 1e3)
        consistent = None
        if world > 1:
            # every rank must hold the same estimate (replicated power iteration on gathered B)
            e_last = torch.tensor([errs[-1][0]], dtype=torch.float64, device=f"cuda:{dev}")
            lo_, hi_ = e_last.clone(), e_last.clone()
            torch.distributed.all_reduce(lo_, op=torch.distributed.ReduceOp.MIN)
            torch.distributed.all_reduce(hi_, op=torch.distributed.ReduceOp.MAX)
            consistent = bool(lo_.item() == hi_.item())
        kt, head, alt = None, None, None
        clocks = clk.summary()
        comm = [solver.comm_bytes(k) for k in range(len(part.sets))]
        sharded_info = {"operands": solver.operands, "exchange_mode": solver.exchange, "panel": solver.layout.panel,
                        "comm_bytes_per_sweep_this_rank": {key: int(sum(c[key] for c in comm)) for key in comm[0]},
                        "nvlink_model_ms_per_sweep": sum(
                            max(c["exchange_out"], c["exchange_in"]) + c["allreduce_top"] + c["allgather_w_in"]
                            for c in comm) / 770e9 * 1e3}
        ttt = None
        if not args.no_ttt:
            solver.init_sigma(guess)
            torch.distributed.barrier()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            n_to_tol = 0
            for n_to_tol in range(1, cfg.max_iterations + 1):
                e, _, _ = sweep()
                fr = solver.frobenius() if cfg.stopping == "frobenius" and e < 1.01 * cfg.tol else None
                if cfg.stopping == "frobenius" and fr is None:
                    continue
                if (fr < cfg.tol) if fr is not None else (e <= cfg.tol):
                    break
            torch.cuda.synchronize()
            t_loop = max_over_ranks(time.perf_counter() - t1, dev)
            ttt = {"seconds": max_over_ranks(setup_s, dev) + t_loop, "sweeps": n_to_tol, "tol": cfg.tol,
                   "stopping": cfg.stopping, "setup_s": setup_s, "timing": "wall, max over ranks"}
        solver.close()
        torch.cuda.empty_cache()

    e2e = None
    if not args.no_e2e and a_host is not None and rank == 0 and world == 1:
        # public API, host buffers: h2d of A, setup, K sweeps, d2h of Σ inside the timed region
        walls = []
        for _ in range(2):   # best of 2: the first call also pays one-time CUDA module/graph set-up
            t0 = time.perf_counter()
            rep = pkg.solve(a_host, part, pkg.IbmiConfig(tol=1e-300, max_iterations=args.steps,
                                                         initial_guess=guess, gemm=args.gemm,
                                                         ozaki_moduli=args.moduli))
            walls.append(time.perf_counter() - t0)
            del rep.result
        wall = min(walls)
        e2e = {"value": args.steps / wall, "unit": "sweeps/s", "walls_s": walls,
               "h2d_bytes_per_step": int(p * p * 8 / args.steps),
               "d2h_bytes_per_step": int(p * p * 8 / args.steps) + 8,
               "note": f"solve(a_host, part, IbmiConfig(max_iterations=steps, gemm={args.gemm!r})) wall time incl. "
                       "A upload, setup, sweeps, per-sweep error readback and Sigma download (best of 2 calls)"}
    if not args.no_e2e and a_host is not None and (world > 1 or args.sharded):
        # public N-rank API (distributed.solve_sharded), host buffers on every rank: h2d of A on
        # each rank, setup, K sweeps, Σ gathered back to host memory; wall time, max over ranks
        from paper_2502_06377_b200.distributed import solve_sharded

        walls = []
        for _ in range(2):
            torch.distributed.barrier()
            t0 = time.perf_counter()
            rep = solve_sharded(a_host, part, pkg.IbmiConfig(tol=1e-300, max_iterations=args.steps,
                                                             initial_guess=guess), exchange=args.exchange,
                                operands=args.operands)
            walls.append(max_over_ranks(time.perf_counter() - t0, dev))
            del rep
        wall = min(walls)
        e2e = {"value": args.steps / wall, "unit": "sweeps/s", "walls_s": walls,
               "h2d_bytes_per_step": int(world * p * p * 8 / args.steps),
               "d2h_bytes_per_step": int(world * p * p * 8 / args.steps),
               "note": "distributed.solve_sharded(a_host, part, IbmiConfig(max_iterations=steps)) on every rank: "
                       "wall time (max over ranks) incl. each rank's A upload, setup, sweeps, per-sweep error "
                       "readback and the Sigma gather to host (best of 2 calls)"}
    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1 and a_host is not None:
        s = cpu_sample(cfg, a_host)
        cpu = {"value": 1.0 / s["sweep_s"], "unit": "sweeps/s", "cores": os.cpu_count(), "kind": "port",
               "sample": s["sample"], "setup_one_set_s": s["setup_one_set_s"], **host_info()}

    def roofline(mode, kt_, igemm_):
        if kt_ is None:
            return None
        if mode == "ozaki":
            ach = igemm_["int8_ops"] / (igemm_["ms"] * 1e-3) / 1e12 if igemm_ and igemm_["ms"] > 0 else None
            pk = int8_peak or INT8_PEAK_TOPS
            return {"bound": "tensor", "kernel": "igemm_tc2_kernel (INT8 residue GEMMs of the Ozaki-II emulation, "
                                                 "tcgen05.mma.cta_group::2 kind::i8, TMA, TMEM)",
                    "achieved": ach, "peak": pk, "unit": "TOPS",
                    "frac": ach / pk if ach else None,
                    "frac_of_nominal": ach / INT8_PEAK_TOPS if ach else None,
                    "traffic": None,
                    "launches_per_sweep": igemm_["launches"] if igemm_ else None,
                    "kernel_ms_per_sweep": igemm_["ms"] if igemm_ else None,
                    "peak_source": ("measured on this box: cuBLASLt int8 GEMM 8192^3 (torch._int_mm), best of 10"
                                    if int8_peak else "nominal B200 dense INT8 (B200_PROFILING.md)") +
                                   "; achieved = algorithmic INT8 ops / CUDA-event time of every igemm launch of a sweep"}
        if p <= 1024 and kt_.get("diag_gemm", 0.0) == 0.0 and kt_.get("estimate_gemm", 0.0) == 0.0:
            # fused small-problem sweep: one cooperative kernel runs every GEMM phase of the sweep
            fl = executed_flops(cfg)
            tf_ = fl / (kt_["panel_gemm"] * 1e-3) / 1e12
            return {"bound": "tensor", "kernel": "small_sweep_kernel (all GEMM phases of a sweep fused: 32x32 DMMA "
                                                 "tiles, operands from L2, grid barriers between phases)",
                    "achieved": tf_, "peak": peak, "unit": "TFLOP/s", "frac": tf_ / peak, "traffic": None,
                    "traffic_note": "operands (A, Sigma, W: 2 MB each at c1) are L2-resident; latency-bound: "
                                    "2K+1 grid barriers and short K loops, not bandwidth or tensor throughput",
                    "peak_source": "measured on this box: DMMA m8n8k4 throughput probe (ibmi_probe_fp64_peak)"}
        panel_flops = sum(2.0 * b * (p - b) ** 2 for b in sizes)
        panel_tf = panel_flops / (kt_["panel_gemm"] * 1e-3) / 1e12
        return {"bound": "tensor", "kernel": "gemm_tma_kernel (panel M = W Sigma_cc, FP64 DMMA, TMA)",
                "achieved": panel_tf, "peak": peak, "unit": "TFLOP/s", "frac": panel_tf / peak,
                **panel_traffic(args.config),
                "peak_source": "measured on this box: DMMA m8n8k4 throughput probe (ibmi_probe_fp64_peak)"}

    if rank == 0:
        tf = flops * sweeps_s / 1e12
        mode = args.gemm if world == 1 and not args.sharded else "dmma"
        line = {
            "metric": "IBMI sweeps/s (FP64) at p=16384" if args.config == "c4" else f"IBMI sweeps/s ({args.config})",
            "value": sweeps_s, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64" if mode == "dmma" else f"f64 via int8 (Ozaki-II, {args.moduli} moduli)",
            "data": "synthetic",
            "config": bench_config(cfg, part),
            "parallelism": f"row-panel sharded x{world}" if world > 1 else "single",
            "gemm": mode,
            "tflops": tf,
            "tflops_frac_of_peak": tf / world / peak,
            "tflops_executed": executed_flops(cfg) * sweeps_s / 1e12,
            "fp64_peak_tflops": peak,
            "int8_peak_tops_measured": int8_peak,
            "setup_s": setup_s,
            "ranks_consistent": consistent,
            "exchange": getattr(solver, "exchange", None) if world > 1 else None,
            "sharded": sharded_info,
            "time_to_tol": ttt,
            "power_iterations": [e[1] for e in errs],
            "error_trace": [e[0] for e in errs],
            "kernel_ms_per_sweep": kt,
            "roofline": roofline(mode, kt, head["igemm"] if head else None) if kt is not None else {
                # the sharded driver has no per-kernel event timing: the whole sweep's executed FLOPs per GPU
                "bound": "tensor", "kernel": "sharded sweep, all FP64 DMMA GEMMs of a rank (gemm_tma_kernel via ibmi_gemm)",
                "achieved": executed_flops(cfg) * sweeps_s / world / 1e12, "peak": peak, "unit": "TFLOP/s",
                "frac": executed_flops(cfg) * sweeps_s / world / 1e12 / peak, "traffic": None,
                "peak_source": "measured on this box: DMMA m8n8k4 throughput probe (ibmi_probe_fp64_peak)"},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "gpu_launches_note": "kernels launched by libibmi_b200.so inside the timed region on rank 0 "
                                 "(graph replays count their kernel nodes)",
            "clocks": clocks,
        }
        if alt is not None:
            line["alt"] = {
                "gemm": alt["mode"], "moduli": args.moduli if alt["mode"] == "ozaki" else None,
                "value": alt["sweeps_s"], "unit": "sweeps/s", "ms_per_step": alt["ms"] / args.steps,
                "tflops": flops * alt["sweeps_s"] / 1e12,
                "tflops_frac_of_fp64_peak": flops * alt["sweeps_s"] / 1e12 / peak,
                "sigma_rel_fro_vs_headline": alt["sigma_rel_fro_vs_headline"],
                "error_trace": [e[0] for e in alt["errs"]],
                "time_to_tol": alt["ttt"], "kernel_ms_per_sweep": alt["kt"],
                "roofline": roofline(alt["mode"], alt["kt"], alt["igemm"]),
                "gpu_launches": int(alt["launches"]), "clocks": alt["clocks"],
                "note": "same context, same Sigma0 and sweep count; Sigma compared after warmup+steps sweeps",
            }
        print(json.dumps(line), file=_JSON_OUT, flush=True)
    if world > 1 or args.sharded:
        torch.distributed.destroy_process_group()


def relaunch(args) -> int:
    """``--gpus N`` outside torchrun: run N ranks under torch.distributed.run on
    this node, or fail (exit 3) when it has fewer than N GPUs."""
    import socket

    import torch

    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs on this node, found {have}; "
              "not running (a multi-GPU number is never measured on fewer GPUs)", file=sys.stderr)
        return 3
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd, stdout=_JSON_OUT.fileno(), stderr=2).returncode


if __name__ == "__main__":
    # The driver reads rank 0's stdout as exactly one JSON line, but NCCL (and
    # anything else in the process) may write to fd 1 -- e.g. "NCCL version ..."
    # at the first collective.  Keep a private copy of stdout for the JSON line
    # and point fd 1 at stderr for everything else.
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    a = parse()
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None and int(ws) != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={ws}; launch with torchrun --nproc-per-node {a.gpus}",
              file=sys.stderr)
        sys.exit(2)
    if a.impl == "reference":
        run_reference(a)
    elif ws is None and a.gpus > 1:
        sys.exit(relaunch(a))
    else:
        run_ours(a)
