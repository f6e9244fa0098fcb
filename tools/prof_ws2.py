import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W, index as I, _lib
k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg2"
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
cl = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
idx = sx.build_index(m, cl, 4096)
if os.environ.get("PROF_EST"):  # the optimizer's walk estimate (enables the prefix exit for short walks)
    print("estimate", sx.estimate_walk_length(idx, m, 0.001, k, seed=w.seed).mean_visited)
if len(sys.argv) > 3:  # timing experiment: SIMDEX_SKIP_EPI mode for the query only
    os.environ["SIMDEX_SKIP_EPI"] = sys.argv[3]
for _ in range(3):
    out = I.query_batch_tensors(idx, m, None, k, True)
torch.cuda.synchronize()
_lib.profile(True)
t = time.perf_counter(); out = I.query_batch_tensors(idx, m, None, k, True); torch.cuda.synchronize()
dt = time.perf_counter() - t
ks = {n: _lib.profile_read(n) for n in ("gemm_topk", "finalize", "walk", "select_rows", "seed_pick", "seed_t0")}
print("k", k, "ms", 1000 * dt, " ".join(f"{n}={v[0]:.3f}ms/{v[1]}" for n, v in ks.items() if v[1]), "stats", _lib.ws_stats(), flush=True)
