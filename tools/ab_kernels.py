"""Per-kernel timing of one serving workload for A/B comparisons of library
builds (SIMDEX_LIB_PATH selects the .so).  Prints one line: the step time
and each main kernel's median per-step milliseconds over --steps steps.

    SIMDEX_LIB_PATH=build/ab/libB.so python tools/ab_kernels.py --config cfg2 --k 10 --steps 30
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _lib, optimizer
from paper_1706_01449_b200 import index as index_mod
from paper_1706_01449_b200 import workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--k", type=int, default=None)
ap.add_argument("--steps", type=int, default=30)
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--prefix-exit", default="auto", choices=["auto", "on", "off"])
a = ap.parse_args()
w = W.CONFIGS[a.config](a.scale) if a.scale != 1.0 else W.CONFIGS[a.config]()
k = a.k or w.k
model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
if a.config in ("cfg1", "cfg3", "cfg5"):
    step = lambda: sx.brute.topk_matmul_tensors(model, k)  # noqa: E731
else:
    plan = optimizer.plan_pipeline(model, k=k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters,
                                   seed=w.seed)
    if a.prefix_exit != "auto":
        index_mod.note_walk_estimate(plan.index, k, 0.0 if a.prefix_exit == "on" else 1e18)
    step = lambda: index_mod.query_batch_tensors(plan.index, model, None, k)  # noqa: E731
for _ in range(3):
    step()
torch.cuda.synchronize()
names = ("gemm_topk", "gemm_topk_prefix", "gemm_topk_full", "finalize", "finalize_prefix", "finalize_full")
per = {n: [] for n in names}
steps = []
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")
for s in range(a.steps):
    flush.fill_(s & 0x7F)
    _lib.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    step()
    e1.record()
    torch.cuda.synchronize()
    steps.append(e0.elapsed_time(e1))
    for n in names:
        ms, c = _lib.profile_read(n)
        if c:
            per[n].append(ms)
    _lib.profile(False)
out = {"lib": os.path.basename(os.environ.get("SIMDEX_LIB_PATH", "default")), "config": a.config, "k": k,
       "prefix_exit": a.prefix_exit, "step_ms": round(statistics.median(steps), 4),
       "pairs": _lib.executed_pairs()}
out.update({n: round(statistics.median(v), 4) for n, v in per.items() if v})
print(json.dumps(out), flush=True)
