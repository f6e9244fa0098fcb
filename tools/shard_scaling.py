"""Per-rank serving time of the multi-GPU partitions, measured one rank at a
time on one GPU (the index path and the blocked product have no collective,
so rank r's step is independent of the others): predicted strong-scaling
efficiency T1 / (N * max_r T_r) for N = 1, 2, 4, 8.
    python tools/shard_scaling.py [cfg] [--graph]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import graphs, index as I, optimizer, sharding
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else "cfg2"
use_graph = "--graph" in sys.argv
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
plan = optimizer.plan_pipeline(m, k=w.k, num_clusters=w.clusters or 8, block_size=4096, max_iters=w.max_iters,
                               seed=w.seed)
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")


def timed(fn, steps=20):
    if use_graph:
        fn = graphs.GraphedCall(fn)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for s in range(steps):
        flush.fill_(s & 0x7F)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


out = {"cfg": cfg, "decision": plan.decision, "graph": use_graph, "ranks": {}}
t1 = None
for n in (1, 2, 4, 8):
    per = []
    for r in range(n):
        if plan.decision == "index":
            if n == 1:
                fn = lambda: I.query_batch_tensors(plan.index, m, None, w.k)  # noqa: E731
            else:
                sh = sharding.IndexShard(plan.index, m, r, n, plan.walk)
                fn = lambda sh=sh: sh.topk_tensors(w.k)  # noqa: E731
        else:
            sh = sharding.UserShard(m, r, n)
            fn = lambda sh=sh: sh.topk_tensors(w.k)  # noqa: E731
        per.append(timed(fn))
    mx = max(per)
    t1 = t1 or mx
    out["ranks"][n] = {"ms": [round(x, 4) for x in per], "max_ms": round(mx, 4),
                       "users_per_s": w.users.shape[0] / (mx / 1e3), "efficiency": t1 / (n * mx)}
print(json.dumps(out))
