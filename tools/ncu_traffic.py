"""DRAM traffic per gemm_topk launch from an ncu --set full capture of
tools/ncu_step.py -> profiles/gemm_topk_traffic.json (read by bench.py's
roofline.traffic, which uses it only while the kernel sources hash to the
value recorded here).

    python tools/ncu_traffic.py gpurun_out/X.ncu-rep --path index|brute [--capture "..."]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

sys.path.insert(0, os.getcwd())
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("--path", default="index")
ap.add_argument("--capture", default="")
ap.add_argument("--out", default=bench.TRAFFIC_FILE)
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--k", type=int, default=10)
a = ap.parse_args()
raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
units = rows[1]
col = {h: i for i, h in enumerate(hdr)}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
launches = {}
order = []
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    if "gemm_topk_kernel" not in name:
        continue
    rd = float(r[col["dram__bytes_read.sum"]]) * scale.get(units[col["dram__bytes_read.sum"]], 1)
    wr = float(r[col["dram__bytes_write.sum"]]) * scale.get(units[col["dram__bytes_write.sum"]], 1)
    order.append((name, rd, wr))
labels = ["gemm_topk_prefix", "gemm_topk_full"] if a.path == "index" else ["gemm_topk"]
for (name, rd, wr), lab in zip(order, labels):
    launches[lab] = {"kernel_name": name, "dram_bytes": rd + wr, "dram_read": rd, "dram_write": wr}
out = {"kernel_source_hash": bench.kernel_source_hash(), "workload": a.workload, "k": a.k, "capture": a.capture or os.path.basename(a.rep),
       "launches": launches}
json.dump(out, open(a.out, "w"), indent=1)
print(json.dumps(out, indent=1))
