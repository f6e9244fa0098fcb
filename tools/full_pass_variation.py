"""Run-to-run variation of the list-order catalogue pass: one process = one
sample; prints the launch times and the operands' device addresses.
python tools/full_pass_variation.py"""
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
step = lambda: I.query_batch_tensors(plan.index, m, None, 10)  # noqa: E731
for _ in range(4):
    step()
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
_lib.profile(True)
for s in range(20):
    flush.fill_(s & 0x7F)
    step()
torch.cuda.synchronize()
out = {}
for name in ("gemm_topk_prefix", "gemm_topk_full", "finalize_prefix", "finalize_full"):
    ms, n = _lib.profile_read(name)
    out[name] = round(ms / max(n, 1), 4)
fl = plan.index._dev.get("full_lists")
ptrs = {"full_b": hex(fl[1][0].data_ptr()) if fl and fl[1] else None,
        "users_pk": hex(_device.packed_users(m.users).data.data_ptr()) if hasattr(_device.packed_users(m.users), "data") else None}
print(out, ptrs, "hashseed", os.environ.get("PYTHONHASHSEED"))
