"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys

path = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/launches.csv"
lines = [l for l in open(path) if l.startswith('"')]
r = csv.reader(lines)
hdr = next(r)
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
for row in r:
    try:
        v = float(row[vi].replace(",", ""))
    except ValueError:
        continue
    v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(row[ui], 1.0)
    name = row[ki].split("(")[0].replace("void ", "").split("<")[0]
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':28s} {'launches':>8s} {'total_ms':>10s} {'share':>6s} {'avg_us':>9s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:28s} {v[0]:8d} {v[1] / 1e3:10.2f} {v[1] / tot:6.3f} {v[1] / v[0]:9.1f}")
print(f"{'TOTAL':28s} {sum(v[0] for v in agg.values()):8d} {tot / 1e3:10.2f}")
