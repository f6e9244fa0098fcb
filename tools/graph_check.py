"""Graph replay of the serving step equals the eager call; timing of both."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import graphs, optimizer, index as I, workloads as W, sharding
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
plan = optimizer.plan_pipeline(m, k=w.k, num_clusters=w.clusters or 8, block_size=4096, max_iters=w.max_iters, seed=w.seed)
if plan.decision == "index":
    fn = lambda: I.query_batch_tensors(plan.index, m, None, w.k)
else:
    fn = lambda: sx.brute.topk_matmul_tensors(m, w.k)[:2]
eager = [t.clone() for t in fn()]
g = graphs.GraphedCall(fn)
out = g()
torch.cuda.synchronize()
same = all(torch.equal(a, b) for a, b in zip(eager, out))
def timeit(f, n=20):
    for _ in range(3): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
print(cfg, "graph == eager:", same, "eager ms %.3f graph ms %.3f" % (timeit(fn), timeit(g)))
# a shard of 1/8 of the users (the 8-GPU per-rank workload), eager vs graph
if plan.decision == "index":
    sh = sharding.IndexShard(plan.index, m, 0, 8, plan.walk)
    f8 = lambda: sh.topk_tensors(w.k)
    g8 = graphs.GraphedCall(f8)
    print("1/8 shard", len(sh.user_ids), "users: eager ms %.3f graph ms %.3f" % (timeit(f8), timeit(g8)))
