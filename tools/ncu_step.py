"""One serving step of a bench workload inside cudaProfilerStart/Stop, for
`ncu --profile-from-start off` (so only the step's kernels are captured).

    ncu --profile-from-start off --set full ... python tools/ncu_step.py --config cfg2 [--k 10]
"""
import argparse
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import index as index_mod
from paper_1706_01449_b200 import optimizer
from paper_1706_01449_b200 import workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg2")
ap.add_argument("--k", type=int, default=None)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
w = W.CONFIGS[a.config]()
k = a.k or w.k
model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
if a.config == "cfg5":
    step = lambda: sx.brute.topk_matmul_tensors(model, k)  # noqa: E731
else:
    plan = optimizer.plan_pipeline(model, k=k, num_clusters=min(w.clusters or 8, w.users.shape[0]),
                                   block_size=4096, max_iters=w.max_iters, seed=w.seed)
    if plan.decision == "index":
        step = lambda: index_mod.query_batch_tensors(plan.index, model, None, k)  # noqa: E731
    else:
        step = lambda: sx.brute.topk_matmul_tensors(model, k)  # noqa: E731
for _ in range(3):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.steps):
    step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ncu_step done", a.config, k)
