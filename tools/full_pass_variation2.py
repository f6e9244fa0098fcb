"""In a process whose list-order catalogue pass is slow: does re-allocating
the full-list operand, or the context arena, change it?
python tools/full_pass_variation2.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _device, _lib, optimizer
from paper_1706_01449_b200 import index as I
from paper_1706_01449_b200 import workloads as W

w = W.CONFIGS["cfg2"]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
plan = optimizer.plan_pipeline(m, k=10, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters, seed=w.seed)
idx = plan.index
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")


def measure(ctx=None, q=None):
    step = lambda: I.query_batch_tensors(idx, m, q, 10, ctx=ctx)  # noqa: E731
    for _ in range(4):
        step()
    torch.cuda.synchronize()
    _lib.profile(True)
    for s in range(10):
        flush.fill_(s & 0x7F)
        step()
    torch.cuda.synchronize()
    ms, n = _lib.profile_read("gemm_topk_full")
    _lib.profile(False)
    return round(ms / max(n, 1), 4)


base = measure()
fresh = []
qs = I.QuerySet(idx, None, q=torch.arange(m.num_users, dtype=torch.int64, device="cuda"))
ctxs = []
for _ in range(3):
    ctxs.append(_lib.Context())
    fresh.append(measure(ctxs[-1].handle, qs))
again = measure()
print("default ctx", base, "fresh contexts", fresh, "default again", again, flush=True)
