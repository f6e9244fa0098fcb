"""One run_pipeline from host matrices after two warm-up runs (for launch lists)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W
w = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"]()
for it in range(3):
    m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    res, rep = sx.run_pipeline(m, k=w.k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters, seed=w.seed)
    _ = res.item_ids
    torch.cuda.synchronize()
print("ok")
