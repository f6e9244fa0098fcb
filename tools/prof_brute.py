import sys, os, time
sys.path.insert(0, os.getcwd())
import torch, numpy as np
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W, _lib, brute
name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
k = int(sys.argv[2]) if len(sys.argv) > 2 else None
scale = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
w = W.CONFIGS[name](scale)
k = k or w.k
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
for _ in range(2):
    ids, sc, h = brute.topk_matmul_tensors(m, k, heap_ops=True)
torch.cuda.synchronize()
_lib.profile(True)
t = time.perf_counter()
ids, sc, h = brute.topk_matmul_tensors(m, k, heap_ops=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
g, _ = _lib.profile_read("gemm_topk"); fz, _ = _lib.profile_read("finalize")
nu, ni, f = w.users.shape[0], w.items.shape[0], w.users.shape[1]
print(f"{name} {nu}x{ni}x{f} k={k}: wall {dt*1e3:.2f} ms gemm {g:.2f} ms finalize {fz:.2f} ms "
      f"-> {nu/dt/1e6:.2f} M users/s, gemm {2*nu*ni*f/g/1e9:.1f} TFLOP/s; appends/user {h.double().mean().item():.1f}", flush=True)
