"""Kernel timeline of one run_pipeline step (bench.py's e2e path) via the
torch profiler (CUPTI): GPU busy time vs wall span, top kernels, largest idle gaps.
python tools/kprof_e2e.py [cfg]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "cfg2"
w = W.CONFIGS[cfg]()
model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
dev = torch.device("cuda", 0)
host_u = torch.from_numpy(model.users.values).pin_memory()
host_i = torch.from_numpy(model.items.values).pin_memory()


def step():
    m2 = sx.ModelPair(sx.FactorMatrix(model.users.values), sx.FactorMatrix(model.items.values))
    m2.users.__dict__["_device"][0] = {"f64": host_u.to(dev, non_blocking=True)}
    m2.items.__dict__["_device"][0] = {"f64": host_i.to(dev, non_blocking=True)}
    res, rep = sx.run_pipeline(m2, k=w.k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters,
                               seed=w.seed, force="index" if cfg != "cfg3" else None)
    _ = res.item_ids
    torch.cuda.synchronize()
    return rep


for _ in range(3):
    step()
t0 = time.perf_counter()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    rep = step()
wall = time.perf_counter() - t0
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
busy = sum(e.time_range.end - e.time_range.start for e in ev)
span = ev[-1].time_range.end - ev[0].time_range.start
print(f"{cfg}: wall {wall * 1e3:.2f} ms (profiled), gpu span {span / 1e3:.2f} ms, gpu busy {busy / 1e3:.2f} ms, "
      f"{len(ev)} device events; stages cluster {rep.cluster_seconds * 1e3:.2f} build {rep.build_seconds * 1e3:.2f} "
      f"est {rep.estimate_seconds * 1e3:.2f} serve {rep.serve_seconds * 1e3:.2f} ms")
agg = {}
for e in ev:
    k = e.name[:70]
    a = agg.setdefault(k, [0.0, 0])
    a[0] += e.time_range.end - e.time_range.start
    a[1] += 1
for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:30]:
    print(f"{t / 1e3:9.3f} ms {c:5d}  {k}")
gaps = []
for a, b in zip(ev, ev[1:]):
    g = b.time_range.start - a.time_range.end
    if g > 0:
        gaps.append((g, a.name[:40], b.name[:40], a.time_range.end - ev[0].time_range.start))
gaps.sort(reverse=True)
print("idle total %.2f ms; largest gaps:" % (sum(g[0] for g in gaps) / 1e3))
for g, a, b, at in gaps[:25]:
    print(f"  {g / 1e3:7.3f} ms at {at / 1e3:7.2f} ms  after {a}  before {b}")
if "--seq" in sys.argv:
    print("timeline (start ms, dur ms, name):")
    t00 = ev[0].time_range.start
    for e in ev:
        print(f"  {(e.time_range.start - t00) / 1e3:8.3f} {(e.time_range.end - e.time_range.start) / 1e3:7.3f}  {e.name[:90]}")
