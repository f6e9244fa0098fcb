import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W, _lib
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
for it in range(2):
    torch.cuda.synchronize(); _lib.profile(True)
    t = time.perf_counter()
    cl = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    t = time.perf_counter(); idx = sx.build_index(m, cl, 4096); torch.cuda.synchronize(); bt = time.perf_counter() - t
    ks = {n: _lib.profile_read(n) for n in ("seed_persistent", "seed_update", "seed_pick", "kmeans_assign", "assign_pack", "gemm_topk", "finalize", "centroid_mean", "bounds")}
    print(f"{cfg} kmeans {dt*1e3:.1f} ms build {bt*1e3:.1f} ms", " ".join(f"{n}={v[0]:.2f}ms/{v[1]}" for n, v in ks.items()), flush=True)
