"""cProfile of run_pipeline (host-side Python cost per function): python tools/cprof_e2e.py [cfg]"""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = W.CONFIGS[cfg]()
model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
dev = torch.device("cuda", 0)
host_u = torch.from_numpy(model.users.values).pin_memory()
host_i = torch.from_numpy(model.items.values).pin_memory()


def step():
    m2 = sx.ModelPair(sx.FactorMatrix(model.users.values), sx.FactorMatrix(model.items.values))
    m2.users.__dict__["_device"][0] = {"f64": host_u.to(dev, non_blocking=True)}
    m2.items.__dict__["_device"][0] = {"f64": host_i.to(dev, non_blocking=True)}
    res, rep = sx.run_pipeline(m2, k=w.k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters,
                               seed=w.seed, force="index" if cfg != "cfg3" else None)
    _ = res.item_ids
    torch.cuda.synchronize()


for _ in range(3):
    step()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(35)
