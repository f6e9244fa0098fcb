"""bench.py's e2e loop with a stage breakdown (profiling off)."""
import sys, os, time
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
for s in range(4):
    m2 = sx.ModelPair(sx.FactorMatrix(model.users.values), sx.FactorMatrix(model.items.values))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    m2.users.__dict__["_device"][0] = {"f64": host_u.to(dev, non_blocking=True)}
    m2.items.__dict__["_device"][0] = {"f64": host_i.to(dev, non_blocking=True)}
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res, rep = sx.run_pipeline(m2, k=w.k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters,
                               seed=w.seed, force="index" if cfg != "cfg3" else None)
    _ = res.item_ids
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st = rep.cluster_seconds + rep.build_seconds + rep.estimate_seconds + rep.serve_seconds
    print(f"{cfg} total {(t2-t0)*1e3:.1f} ms h2d {(t1-t0)*1e3:.1f} pipeline {(t2-t1)*1e3:.1f} stages {st*1e3:.1f}: "
          f"cluster {rep.cluster_seconds*1e3:.1f} build {rep.build_seconds*1e3:.1f} est {rep.estimate_seconds*1e3:.1f} "
          f"serve {rep.serve_seconds*1e3:.1f}", flush=True)
