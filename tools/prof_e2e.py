import sys, os, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W, _lib
w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]()
for it in range(3):
    m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    torch.cuda.synchronize()
    _lib.profile(True)
    t = time.perf_counter()
    if it == 2:
        pr = cProfile.Profile(); pr.enable()
    res, rep = sx.run_pipeline(m, k=w.k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters, seed=w.seed)
    ids = res.item_ids
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    if it == 2:
        pr.disable()
    print(f"iter {it}: total {dt*1000:.1f} ms  " + " ".join(f"{k}={v:.4f}" for k, v in
          [("cluster", rep.cluster_seconds), ("build", rep.build_seconds), ("est", rep.estimate_seconds), ("serve", rep.serve_seconds)]), rep.decision, flush=True)
    for name in ("kmeans_assign", "seed_update", "centroid_mean", "walk", "gemm_topk", "finalize", "bounds"):
        ms, n = _lib.profile_read(name)
        print(f"   {name}: {ms:.2f} ms x{n}")
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
