import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
cl = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
torch.cuda.synchronize()
print("ok", cfg)
