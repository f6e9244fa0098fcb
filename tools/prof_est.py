"""Where estimate_walk_length's time goes (cProfile + per-kernel events)."""
import sys, os, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W, optimizer as O, _lib
w = W.CONFIGS["cfg2"]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
cl = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
idx = sx.build_index(m, cl, 4096)
for it in range(4):
    torch.cuda.synchronize()
    if it == 3:
        _lib.profile(True)
        pr = cProfile.Profile(); pr.enable()
    t = time.perf_counter()
    est = O.estimate_walk_length(idx, m, 0.001, w.k, seed=w.seed)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    if it == 3:
        pr.disable()
    print(f"estimate {dt*1e3:.2f} ms mean {est.mean_visited:.1f}", flush=True)
for n in ("gemm_topk", "finalize", "walk"):
    print(n, _lib.profile_read(n))
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
