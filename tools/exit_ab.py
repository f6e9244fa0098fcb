import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W, index as I, _lib
w = W.CONFIGS[sys.argv[1]]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
cl = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
idx = sx.build_index(m, cl, 4096)
for k in [int(x) for x in sys.argv[2:]]:
    est = sx.estimate_walk_length(idx, m, 0.001, k, seed=w.seed).mean_visited
    for mode in ("off", "on"):
        I.note_walk_estimate(idx, k, 0.0 if mode == "on" else 1e9)
        for _ in range(3):
            I.query_batch_tensors(idx, m, None, k, True)
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t = time.perf_counter(); I.query_batch_tensors(idx, m, None, k, True); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
        print(f"{sys.argv[1]} K={k} est={est:.0f} ({est/4096:.2f} B) exit {mode}: {1000*min(ts):.3f} ms", flush=True)
