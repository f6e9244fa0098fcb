"""Per-stage kernel breakdown of run_pipeline's pieces (cluster, build,
estimate, serve), each run alone under the torch profiler after warm-up.
python tools/kprof_stages.py [cfg]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import optimizer as O
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = W.CONFIGS[cfg]()
model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))


def stages():
    cl = sx.kmeans(model.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
    yield "cluster", cl
    idx = sx.build_index(model, cl, 4096)
    yield "build", idx
    est = O.estimate_walk_length(idx, model, O.DEFAULT_SAMPLE_FRACTION, w.k, w.seed)
    yield "estimate", est
    res = sx.query_batch(idx, model, None, w.k, work_sharing=True, precomputed=est.sampled)
    _ = res.item_ids
    yield "serve", res


for _ in range(3):
    for _ in stages():
        torch.cuda.synchronize()
gen = stages()
while True:
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        try:
            name, _ = next(gen)
        except StopIteration:
            break
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    if not ev:
        continue
    ev.sort(key=lambda e: e.time_range.start)
    busy = sum(e.time_range.end - e.time_range.start for e in ev)
    span = ev[-1].time_range.end - ev[0].time_range.start
    print(f"== {name}: span {span / 1e3:.3f} ms busy {busy / 1e3:.3f} ms, {len(ev)} events")
    agg = {}
    for e in ev:
        a = agg.setdefault(e.name[:80], [0.0, 0])
        a[0] += e.time_range.end - e.time_range.start
        a[1] += 1
    for k, (t, c) in sorted(agg.items(), key=lambda x: -x[1][0])[:14]:
        print(f"   {t / 1e3:8.3f} ms {c:4d}  {k}")
