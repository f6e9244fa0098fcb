"""Kernel timeline of one rank's serving step at N ranks (CUPTI via the torch
profiler): every kernel/copy with its duration and the idle gap before it.
python tools/kprof_shard.py [cfg] [N] [rank]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import index as I, optimizer, sharding
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
r = int(sys.argv[3]) if len(sys.argv) > 3 else 0
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
plan = optimizer.plan_pipeline(m, k=w.k, num_clusters=w.clusters or 8, block_size=4096, max_iters=w.max_iters,
                               seed=w.seed)
if n == 1:
    fn = lambda: I.query_batch_tensors(plan.index, m, None, w.k)  # noqa: E731
else:
    sh = sharding.IndexShard(plan.index, m, r, n, plan.walk)
    fn = lambda: sh.topk_tensors(w.k)  # noqa: E731
for _ in range(3):
    fn()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fn()
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA),
            key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
prev = t0
for e in ev:
    print(f"{(e.time_range.start - t0) / 1e3:8.3f} ms  gap {(e.time_range.start - prev) / 1e3:6.3f}  "
          f"dur {(e.time_range.end - e.time_range.start) / 1e3:6.3f}  {e.name[:80]}")
    prev = e.time_range.end
print(f"span {(ev[-1].time_range.end - t0) / 1e3:.3f} ms, busy {sum(e.time_range.end - e.time_range.start for e in ev) / 1e3:.3f} ms")
