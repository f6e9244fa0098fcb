"""Top stall SASS lines of an ncu report: python tools/ncu_sass_hot.py rep [N]"""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
si = h.index("Warp Stall Sampling (All Samples)")
rows = [x for x in r[2:] if len(x) > si]
tot = sum(int(x[si]) for x in rows if x[si].isdigit())
order = sorted(range(len(rows)), key=lambda i: -int(rows[i][si]) if rows[i][si].isdigit() else 0)
for i in order[:n]:
    x = rows[i]
    print(f"{int(x[si]):6d} {100*int(x[si])/tot:5.1f}%  [{i:4d}] {x[1].strip()[:80]}")
