"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, collections, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ki, vi, ui = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Unit')
scale = {'nsecond': 1e-6, 'ns': 1e-6, 'usecond': 1e-3, 'us': 1e-3, 'msecond': 1.0, 'ms': 1.0}
agg = collections.OrderedDict()
seq = []
for r in data:
    name = r[ki].split('(')[0]
    v = float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    agg.setdefault(name, [0, 0.0])
    agg[name][0] += 1
    agg[name][1] += v
    seq.append((name, v))
tot = sum(v for _, v in seq)
print(f"| kernel | launches | total ms | share |\n|---|---|---|---|")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {n} | {t:.3f} | {100 * t / tot:.1f}% |")
print(f"| **total** | {len(seq)} | {tot:.3f} | 100% |")
if len(sys.argv) > 2:
    for n, v in seq[:int(sys.argv[2])]:
        print(f"  {n:40s} {v:.3f}")
