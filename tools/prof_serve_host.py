"""Host-side cost of query_batch (the serve stage of run_pipeline)."""
import sys, os, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W, index as I, optimizer as O
w = W.CONFIGS["cfg2"]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
cl = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
idx = sx.build_index(m, cl, 4096)
est = O.estimate_walk_length(idx, m, 0.001, w.k, seed=w.seed)
for it in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    if it == 3:
        pr = cProfile.Profile(); pr.enable()
    r = I.query_batch(idx, m, None, w.k, work_sharing=True, precomputed=est.sampled)
    torch.cuda.synchronize()
    if it == 3:
        pr.disable()
    print(f"query_batch {1e3*(time.perf_counter()-t):.2f} ms", flush=True)
pstats.Stats(pr).sort_stats("tottime").print_stats(15)
