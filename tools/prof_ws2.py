import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W, index as I
k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
w = W.cfg2()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
cl = sx.kmeans(m.users, 256, max_iters=3, seed=1)
idx = sx.build_index(m, cl, 4096)
for _ in range(3):
    out = I.query_batch_tensors(idx, m, None, k, True)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("timed")
t = time.perf_counter(); out = I.query_batch_tensors(idx, m, None, k, True); torch.cuda.synchronize()
print("k", k, "ms", 1000 * (time.perf_counter() - t), flush=True)
