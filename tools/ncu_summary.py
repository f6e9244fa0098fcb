"""Summarise an ncu report: headline metrics per kernel and the top SASS
stall sites.  usage: python tools/ncu_summary.py report.ncu-rep [top_n]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top_n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed.avg.per_cycle_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_bytes.sum"]
idx = {w: h.index(w) for w in want if w in h}
units = rows[1]
for r in rows[2:]:
    print("kernel:", r[idx["Kernel Name"]][:100])
    for w, i in idx.items():
        if w != "Kernel Name":
            print(f"  {w:90s} {r[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        blocks.append((r[1], cur))
        continue
    if cur is not None:
        cur.append(r)
for name, b in blocks:
    hh = b[0]
    data = [dict(zip(hh, x)) for x in b[1:] if len(x) == len(hh)]
    tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data) or 1.0
    ex = sum(float(d["Instructions Executed"] or 0) for d in data)
    print(f"top stall sites of {name[:80]} (warp-instructions executed {ex:.3e})")
    for d in sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[:top_n]:
        print(f"  {100 * float(d['Warp Stall Sampling (All Samples)']) / tot:5.1f}%  exec={d['Instructions Executed']:>10}  {d['Source'][:80]}")
