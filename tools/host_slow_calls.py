"""Host-side slow calls inside one run_pipeline pass: every torch.empty and
library call taking more than 30 us, with its offset from the pass start.
python tools/host_slow_calls.py [cfg]"""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _lib, workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
w = W.CONFIGS[cfg]()
model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
dev = torch.device("cuda", 0)
host_u = torch.from_numpy(model.users.values).pin_memory()
host_i = torch.from_numpy(model.items.values).pin_memory()
LOG = []
T0 = [0.0]


def wrap(fn, label):
    def inner(*a, **k):
        t = time.perf_counter()
        r = fn(*a, **k)
        d = time.perf_counter() - t
        if d > 30e-6:
            what = label(a, k) if callable(label) else label
            LOG.append((t - T0[0], d, what))
        return r
    return inner


torch.empty = wrap(torch.empty, lambda a, k: f"torch.empty{tuple(a[0]) if a and not isinstance(a[0], int) else a} {k.get('dtype')}")
_lib.call = wrap(_lib.call, lambda a, k: f"lib.{a[0]}")
torch.Tensor.item = wrap(torch.Tensor.item, "tensor.item")
torch.Tensor.tolist = wrap(torch.Tensor.tolist, "tensor.tolist")
torch.cuda.synchronize = wrap(torch.cuda.synchronize, "cuda.synchronize")
torch.cuda.Stream.synchronize = wrap(torch.cuda.Stream.synchronize, "stream.synchronize")
torch.Tensor.to = wrap(torch.Tensor.to, "tensor.to")
torch.Tensor.copy_ = wrap(torch.Tensor.copy_, "tensor.copy_")


def step():
    m2 = sx.ModelPair(sx.FactorMatrix(model.users.values), sx.FactorMatrix(model.items.values))
    torch.cuda.synchronize()
    T0[0] = time.perf_counter()
    LOG.clear()
    m2.users.__dict__["_device"][0] = {"f64": host_u.to(dev, non_blocking=True)}
    m2.items.__dict__["_device"][0] = {"f64": host_i.to(dev, non_blocking=True)}
    res, rep = sx.run_pipeline(m2, k=w.k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters,
                               seed=w.seed, force="index" if cfg != "cfg3" else None)
    _ = res.item_ids
    torch.cuda.synchronize()
    return time.perf_counter() - T0[0]


import gc
gc.collect()
for i in range(4):
    st0 = torch.cuda.memory_stats()
    step()
    st1 = torch.cuda.memory_stats()
    print(f"pass {i}: cudaMalloc calls {st1.get('segment.all.allocated', 0) - st0.get('segment.all.allocated', 0)}, cudaFree "
          f"{st1.get('segment.all.freed', 0) - st0.get('segment.all.freed', 0)}, reserved {st1.get('reserved_bytes.all.current', 0) >> 20} MiB, "
          f"allocated {st1.get('allocated_bytes.all.current', 0) >> 20} MiB, gc garbage {gc.collect()}")
t = step()
print(f"pass {t * 1e3:.2f} ms; calls over 30 us (offset ms, dur ms):")
for at, d, what in LOG:
    print(f"  {at * 1e3:8.3f} {d * 1e3:7.3f}  {what}")
