"""Per-kernel times of one rank's serving step at N ranks (index path,
cluster-routed users), measured alone on one GPU:
python tools/shard_kernels.py [cfg] [N] [rank]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _lib, index as I, optimizer, sharding
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
steps = 20
_lib.profile(True)
ts = []
for s in range(steps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
out = {"cfg": cfg, "n": n, "rank": r, "step_ms": statistics.median(ts), "stats": list(_lib.ws_stats())}
for name in ("gemm_topk_prefix", "gemm_topk_full", "finalize_prefix", "finalize_full", "walk"):
    ms, cnt = _lib.profile_read(name)
    if cnt:
        out[name] = round(ms / steps, 4)
_lib.profile(False)
print(json.dumps(out))
