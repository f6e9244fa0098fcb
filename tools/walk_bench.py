"""Walk kernel timing (Algorithm 1, query_batch work_sharing=False): a batch
of users through simdex_walk32 (throughput, achieved bytes/s over the
algorithmic 4f+8 bytes per visited entry) and single-query latency (the
query_user path).  python tools/walk_bench.py [cfg] [k]"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _device, _lib, _ops
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
cl = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
idx = sx.build_index(m, cl, 4096)
f = m.factors
rng = np.random.default_rng(0)
q = np.sort(rng.choice(m.num_users, 20000, replace=False))
qt = torch.as_tensor(q, device="cuda")
qc = idx.device_assignment().index_select(0, qt).to(torch.int32)
ids, bounds = idx.device_lists()
args = (_device.f64(m.users), _device.norms(m.users), _device.f64(m.items), ids, bounds, qt, qc, k)
import inspect
kw = dict(users32=_device.f32_exact(m.users), items32=_device.f32_exact(m.items)) if "users32" in inspect.signature(_ops.walk).parameters else {}
for _ in range(2):
    out = _ops.walk(*args, **kw)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
out = _ops.walk(*args, **kw)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
vis = out[2].cpu().numpy()
alg_bytes = float(vis.sum()) * (4 * f + 8)
# single-query latency through the public API
lat = []
for u in q[:200]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sx.query_user(idx, m, int(u), k)
    lat.append(time.perf_counter() - t0)
print(json.dumps({"lib": os.path.basename(os.environ.get("SIMDEX_LIB_PATH", "default")), "cfg": cfg, "k": k,
                  "batch_users": len(q), "batch_ms": round(ms, 3), "mean_visited": float(vis.mean()),
                  "users_per_s": len(q) / (ms / 1e3), "alg_GBps": alg_bytes / (ms / 1e3) / 1e9,
                  "query_user_ms_median": round(1e3 * float(np.median(lat)), 3)}), flush=True)
