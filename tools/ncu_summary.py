"""Summarise an ncu launch-list CSV and a --set full report into markdown.

    python tools/ncu_summary.py <launches.csv> <full.ncu-rep> <out.md> [title]
"""
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "launch__cluster_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct",
    "smsp__warp_issue_stalled_wait_per_warp_active.pct",
    "smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct",
    "smsp__warp_issue_stalled_not_selected_per_warp_active.pct",
    "smsp__warp_issue_stalled_selected_per_warp_active.pct",
    "smsp__warp_issue_stalled_dispatch_stall_per_warp_active.pct",
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            v = float(d["Metric Value"].replace(",", ""))
            unit = d["Metric Unit"]
            v = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v
            out.append((d["Kernel Name"], v))
    return out


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for i, n in enumerate(hdr):
            if n in METRICS:
                d[n] = (r[i], units[i])
        res.append((r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?", d))
    return res


def main():
    lcsv, rep, out = sys.argv[1:4]
    title = sys.argv[4] if len(sys.argv) > 4 else "ncu summary"
    L = launches(lcsv)
    tot = sum(v for _, v in L)
    agg = {}
    for n, v in L:
        key = n.split("(")[0][:70]
        agg.setdefault(key, [0, 0.0])
        agg[key][0] += 1
        agg[key][1] += v
    lines = [f"# {title}", "",
             "## Launch list (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised)", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| `{k}` | {c} | {v:.3f} | {100 * v / tot:.1f}% |")
    lines += [f"| **total** | {len(L)} | {tot:.3f} | 100% |", "", "Per launch:", "", "| # | kernel | ms |",
              "|---|---|---|"]
    for i, (n, v) in enumerate(L):
        lines.append(f"| {i} | `{n[:70]}` | {v:.3f} |")
    if rep != "-":
        for name, d in full(rep):
            lines += ["", f"## ncu --set full: `{name[:90]}`", "", "| metric | value | unit |", "|---|---|---|"]
            for m in METRICS:
                if m in d:
                    lines.append(f"| {m} | {d[m][0]} | {d[m][1]} |")
    open(out, "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
