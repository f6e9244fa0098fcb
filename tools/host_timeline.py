"""Host-side timeline of one run_pipeline step as bench.py's e2e runs it
(pinned host buffers, non-blocking H2D): every library call, host read
(item / tolist / cpu / stream sync) and pinned staging, with wall stamps, so
the GPU idle gaps of tools/kprof_e2e.py can be matched to host work.
python tools/host_timeline.py [cfg] [min_ms]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _lib, _ops
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
min_ms = float(sys.argv[2]) if len(sys.argv) > 2 else 0.02
w = W.CONFIGS[cfg]()
model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
dev = torch.device("cuda", 0)
host_u = torch.from_numpy(model.users.values).pin_memory()
host_i = torch.from_numpy(model.items.values).pin_memory()
log, t0 = [], [0.0]


def wrap(obj, name, label):
    orig = getattr(obj, name)

    def f(*a, **k):
        t = time.perf_counter()
        r = orig(*a, **k)
        log.append((t - t0[0], time.perf_counter() - t, label + (f":{a[0]}" if label == "call" and a else "")))
        return r
    setattr(obj, name, f)


wrap(_lib, "call", "call")
_ops.call = _lib.call
for nm in ("item", "tolist", "cpu", "pin_memory"):
    wrap(torch.Tensor, nm, nm)
wrap(torch.cuda.Stream, "synchronize", "stream.sync")
wrap(torch.cuda, "synchronize", "cuda.sync")


def step():
    m2 = sx.ModelPair(sx.FactorMatrix(model.users.values), sx.FactorMatrix(model.items.values))
    torch.cuda.synchronize()
    log.clear()
    t0[0] = time.perf_counter()
    m2.users.__dict__["_device"] = {0: {"f64": host_u.to(dev, non_blocking=True)}}
    m2.items.__dict__["_device"] = {0: {"f64": host_i.to(dev, non_blocking=True)}}
    res, rep = sx.run_pipeline(m2, k=w.k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters,
                               seed=w.seed, force="index" if cfg != "cfg3" else None)
    _ = res.item_ids
    torch.cuda.synchronize()
    return time.perf_counter() - t0[0], rep


for _ in range(3):
    total, rep = step()
print(f"{cfg}: step {total * 1e3:.2f} ms; stages cluster {rep.cluster_seconds * 1e3:.2f} build "
      f"{rep.build_seconds * 1e3:.2f} est {rep.estimate_seconds * 1e3:.2f} serve {rep.serve_seconds * 1e3:.2f}")
prev_end = 0.0
for ts, dur, what in log:
    gap = ts - prev_end
    if dur * 1e3 >= min_ms or gap * 1e3 >= 0.1:
        print(f"{ts * 1e3:8.3f} ms  +{gap * 1e3:6.3f} host  {dur * 1e3:7.3f} ms  {what}")
    prev_end = ts + dur
