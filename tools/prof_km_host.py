"""Where k-means wall time goes (cProfile; GPU waits show up in .item()/.cpu())."""
import sys, os, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
for it in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    if it == 2:
        pr = cProfile.Profile(); pr.enable()
    cl = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
    torch.cuda.synchronize()
    if it == 2:
        pr.disable()
    print(f"kmeans {1e3*(time.perf_counter()-t):.1f} ms", flush=True)
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
