"""Where CTA 0 of gemm_topk spends its cycles (diagnostic build:
make EXTRA=-DSIMDEX_EPI_TIMING=1 OBJDIR=../../build/ab/objE LIB=../../build/ab/libE.so;
SIMDEX_LIB_PATH=build/ab/libE.so python tools/epi_timing.py [cfg] [k]).  Every
gemm launch of one serving step adds into the same counters."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _lib, optimizer
from paper_1706_01449_b200 import index as I
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
if cfg in ("cfg3", "cfg5", "cfg1"):
    step = lambda: sx.brute.topk_matmul_tensors(m, k)  # noqa: E731
else:
    plan = optimizer.plan_pipeline(m, k=k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters,
                                   seed=w.seed)
    step = lambda: I.query_batch_tensors(plan.index, m, None, k)  # noqa: E731
lib = _lib.load()
buf = (C.c_ulonglong * 16)()
step()
torch.cuda.synchronize()
lib.simdex_dbg_epi_timing(buf)
step()
torch.cuda.synchronize()
lib.simdex_dbg_epi_timing(buf)
v = list(buf)
tiles = max(v[3], 1)
tot = v[0] + v[1] + v[2]
print(f"{cfg} k={k}: epilogue warp 2 of CTA 0 over {v[3]} tiles: per tile {tot / tiles:.0f} cycles = wait full "
      f"{v[0] / tiles:.0f} + TMEM loads {v[1] / tiles:.0f} + processing {v[2] / tiles:.0f}")
mt = max(v[7], 1)
print(f"  processing cycles by tile place in the unit: t=0 {v[9]}, 1-3 {v[10]}, 4-7 {v[11]}, >=8 {v[12]} "
      f"(shares {v[9] / max(v[2], 1):.2f} / {v[10] / max(v[2], 1):.2f} / {v[11] / max(v[2], 1):.2f} / {v[12] / max(v[2], 1):.2f})")
print(f"  MMA warp over {v[7]} tiles: per tile wait empty accumulator {v[5] / mt:.0f}, wait operand stage "
      f"{v[6] / mt:.0f} cycles; producer wait for an empty stage {v[8] / mt:.0f} cycles per tile")
