"""Top CUDA source lines by warp-stall samples: python tools/ncu_src_hot.py rep [N] [kernel-substring]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
ksub = sys.argv[3] if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_fn, agg = None, {}
si = None
for r in rows:
    if len(r) >= 2 and r[0] == "Function Name":
        cur_fn = r[1]
        continue
    if len(r) > 4 and r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if si is None or len(r) <= si or not r[0]:
        continue
    if ksub and (cur_fn is None or ksub not in cur_fn):
        continue
    try:
        v = int(r[si])
    except ValueError:
        continue
    key = (r[0], r[1][:100])
    agg[key] = agg.get(key, 0) + v
tot = sum(agg.values()) or 1
for (ln, src), v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
    print(f"{v:7d} {100 * v / tot:5.1f}%  L{ln:>5}  {src}")
