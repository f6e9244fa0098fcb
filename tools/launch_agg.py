"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel.
usage: python tools/launch_agg.py launches.csv [top_n]"""
import csv, collections, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[1:]:
    if len(r) <= vi or r[0] == "ID":
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    v = float(r[vi].replace(",", ""))
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1e-3)
    a = agg.setdefault(name, [0.0, 0])
    a[0] += v * scale
    a[1] += 1
tot = sum(a[0] for a in agg.values())
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
print(f"{'kernel':60s} {'us':>10s} {'launches':>8s} {'share':>6s}")
for name, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
    print(f"{name[:60]:60s} {v:10.1f} {c:8d} {100 * v / tot:5.1f}%")
print(f"{'total':60s} {tot:10.1f}")
