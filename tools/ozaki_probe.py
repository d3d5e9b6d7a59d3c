"""Ozaki-II emulated FP64 GEMM: accuracy against a long-double reference and
DMMA, throughput at the c4 panel shape, and c4 sweeps with the panel GEMM
emulated (error trace / Σ against the FP64 DMMA run)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2502_06377_b200 as pkg
from paper_2502_06377_b200 import _abi, linalg

L = _abi.lib()
dev = torch.device("cuda:0")


def ref_ld(x, y):
    return (x.astype(np.longdouble) @ y.astype(np.longdouble).T)


def accuracy():
    rng = np.random.default_rng(0)
    cases = []
    m, n, k = 256, 384, 2048
    cases.append(("gauss", rng.standard_normal((m, k)), rng.standard_normal((n, k))))
    cases.append(("wide-range rows", rng.standard_normal((m, k)) * np.exp(rng.uniform(-20, 20, (m, 1))),
                  rng.standard_normal((n, k)) * np.exp(rng.uniform(-20, 20, (n, 1)))))
    cases.append(("wide-range entries", rng.standard_normal((m, k)) * np.exp(rng.uniform(-8, 8, (m, k))),
                  rng.standard_normal((n, k)) * np.exp(rng.uniform(-8, 8, (n, k)))))
    cases.append(("odd sizes", rng.standard_normal((131, 1001)), rng.standard_normal((517, 1001))))
    for name, x, y in cases:
        r = ref_ld(x, y)
        scale = np.abs(x).astype(np.longdouble) @ np.abs(y).astype(np.longdouble).T
        xd = torch.from_numpy(x).to(dev)
        yd = torch.from_numpy(y).to(dev)
        cd = linalg.dgemm_nt(xd, yd).cpu().numpy()
        e_d = float(np.max(np.abs(cd - r) / scale))
        line = [f"{name:20s} dmma {e_d:.2e}"]
        for nm in (12, 14, 16, 18, 20):
            co = linalg.dgemm_nt_ozaki(xd, yd, nm).cpu().numpy()
            e_o = float(np.max(np.abs(co - r) / scale))
            line.append(f"oz{nm} {e_o:.2e}")
        print("  ".join(line), flush=True)


def timing():
    from paper_2502_06377_b200 import configs
    m, n, k = 2560, 14080, 14080
    x = torch.randn(m, k, dtype=torch.float64, device=dev)
    y = torch.randn(n, k, dtype=torch.float64, device=dev)
    for nm in (14, 16, 18, 20):
        linalg.dgemm_nt_ozaki(x, y, nm)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            linalg.dgemm_nt_ozaki(x, y, nm)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 3
        print(f"panel shape {m}x{n}x{k} oz{nm}: {dt*1e3:.2f} ms  {2*m*n*k/dt/1e12:.1f} TFLOP/s-equivalent", flush=True)
    c0 = linalg.dgemm_nt(x, y)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        linalg.dgemm_nt(x, y)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    print(f"panel shape dmma: {dt*1e3:.2f} ms  {2*m*n*k/dt/1e12:.1f} TFLOP/s", flush=True)


def sweeps(name="c3", nsweeps=12, moduli=(16, 18)):
    from paper_2502_06377_b200 import configs
    from paper_2502_06377_b200.device import DeviceSolver
    cfg = configs.get_config(name)
    a = torch.as_tensor(configs.make_matrix(name), device=dev)
    runs = {}
    for nm in (0,) + tuple(moduli):
        _abi.check(L.ibmi_tune(7, nm))
        ds = DeviceSolver(a, partition=cfg.partition())
        ds.setup()
        ds.init_sigma(1 if cfg.guess == "jacobi" else 0)
        errs, ts = [], []
        for it in range(nsweeps):
            e, pi, conv = ds.sweep(1e-9, 5000)
            errs.append(e)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for it in range(3):
            ds.sweep(1e-9, 5000)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 3
        sig = ds.sigma(on_device=True).clone()
        print("   timed:", {k: round(v, 2) for k, v in ds.sweep_timed(1e-9, 5000)[3].items()}, flush=True)
        fr = ds.frobenius()
        ds.close()
        runs[nm] = (errs, sig, dt, fr)
        print(f"{name} moduli={nm}: {1/dt:.2f} sweeps/s  frob={fr:.3e}  errs={['%.3e' % x for x in errs[-4:]]}", flush=True)
    _abi.check(L.ibmi_tune(7, 0))
    e0, s0, _, _ = runs[0]
    for nm in moduli:
        e1, s1, _, _ = runs[nm]
        rel = float(torch.linalg.norm(s1 - s0) / torch.linalg.norm(s0))
        de = max(abs(x - y) / max(abs(x), 1e-300) for x, y in zip(e0, e1))
        print(f"{name} moduli={nm}: Sigma rel-fro vs DMMA {rel:.3e}; max rel err-trace diff {de:.3e}", flush=True)


if __name__ == "__main__":
    what = sys.argv[1:] or ["accuracy", "timing"]
    if "accuracy" in what:
        accuracy()
    if "timing" in what:
        timing()
    for w in what:
        if w.startswith("chunks:"):
            from paper_2502_06377_b200 import configs
            from paper_2502_06377_b200.device import DeviceSolver
            nm = w.split(":")[1]
            cfg = configs.get_config(nm)
            a = torch.as_tensor(configs.make_matrix(nm), device=dev)
            for ch, pair in ((1, 0), (1, 1), (4, 1)):
                _abi.check(L.ibmi_tune(10, ch))
                _abi.check(L.ibmi_tune(11, pair))
                ds = DeviceSolver(a, partition=cfg.partition())
                ds.set_emulation(16)
                ds.setup()
                ds.init_sigma(0)
                for _ in range(2):
                    ds.sweep(1e-9, 5000)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                for _ in range(4):
                    ds.sweep(1e-9, 5000)
                torch.cuda.synchronize()
                dt = (time.perf_counter() - t0) / 4
                tm = ds.sweep_timed(1e-9, 5000)[3]
                print(f"chunks={ch} pair={pair}: {1/dt:.2f} sweeps/s (graph), timed {dict((k, round(v, 2)) for k, v in tm.items())}", flush=True)
                ds.close()
            _abi.check(L.ibmi_tune(10, 1))
            _abi.check(L.ibmi_tune(11, 1))
        if w.startswith("profile:"):
            _, nm, mod = w.split(":")
            from paper_2502_06377_b200 import configs
            from paper_2502_06377_b200.device import DeviceSolver
            cfg = configs.get_config(nm)
            a = torch.as_tensor(configs.make_matrix(nm), device=dev)
            _abi.check(L.ibmi_tune(7, int(mod)))
            ds = DeviceSolver(a, partition=cfg.partition())
            ds.setup()
            ds.init_sigma(1 if cfg.guess == "jacobi" else 0)
            ds.sweep(1e-9, 5000)
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
            ds.sweep(1e-9, 5000)
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
        if w.startswith("sweeps:"):
            _, nm, ns = w.split(":")
            sweeps(nm, int(ns))
