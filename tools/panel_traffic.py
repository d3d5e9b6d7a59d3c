"""DRAM traffic of the panel GEMM per config from an ncu metric CSV.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --profile-from-start off -k regex:gemm_tma --csv \
        --log-file gpurun_out/traffic_c4.csv python tools/profile_sweep.py --config c4
    python tools/panel_traffic.py c4=gpurun_out/traffic_c4.csv c3=... > profiles/r02_panel_traffic.json

One eager sweep launches gemm_tma_kernel in the order K1, K2 per set, then the
estimate and Gram GEMMs: the panel GEMM (K1) is every second launch of the
first 2K.  bench.py reads the JSON for `roofline.traffic` (bytes per launch,
mean over the K panel launches of a sweep)."""
import collections
import csv
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_06377_b200 import configs  # noqa: E402

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1.0}
out = {}
for arg in sys.argv[1:]:
    name, path = arg.split("=", 1)
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ii, ki, mi, vi, ui = (hdr.index(k) for k in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    launches = collections.OrderedDict()
    for r in data:
        if "gemm_tma" not in r[ki]:
            continue
        launches.setdefault(r[ii], {})[r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    seq = list(launches.values())
    cfg = configs.get_config(name)
    sizes = [len(s) for s in cfg.partition().sets]
    k = len(sizes)
    panel = seq[0:2 * k:2]
    assert len(panel) == k, (name, len(seq))
    rd = [x["dram__bytes_read.sum"] for x in panel]
    wr = [x["dram__bytes_write.sum"] for x in panel]
    tm = [x["gpu__time_duration.sum"] for x in panel]
    p = cfg.p
    algo = [8.0 * (b * (p - b) + (p - b) ** 2 + 2 * b * (p - b)) for b in sizes]   # W + Σ_cc read, M written twice
    out[name] = {"bytes_per_launch": (sum(rd) + sum(wr)) / k, "read_per_launch": sum(rd) / k,
                 "write_per_launch": sum(wr) / k, "algorithmic_bytes_per_launch": sum(algo) / k,
                 "panel_launches": k, "ncu_ms_per_launch": 1e3 * sum(tm) / k,
                 "source": os.path.basename(path),
                 "how": "ncu dram__bytes_read.sum + dram__bytes_write.sum of the K panel-GEMM launches "
                        "(gemm_tma_kernel, every second launch of the first 2K) of one eager sweep, mean per launch; "
                        "split-K partial tiles are in the write figure, splitk_reduce_kernel is a separate launch"}
print(json.dumps(out, indent=1))
