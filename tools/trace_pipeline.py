"""Trace run_pipeline: every library call and host sync with wall-clock stamps."""
import sys, os, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W, _lib
w = W.CONFIGS["cfg2"]()
log = []
t0 = [0.0]
orig_call = _lib.call
def call(name, *a):
    t = time.perf_counter()
    r = orig_call(name, *a)
    log.append(("call", name, t - t0[0], time.perf_counter() - t))
    return r
_lib.call = call
import paper_1706_01449_b200._ops as _ops
_ops.call = call
orig_item = torch.Tensor.item
def item(self):
    t = time.perf_counter(); r = orig_item(self); log.append(("item", "", t - t0[0], time.perf_counter() - t)); return r
torch.Tensor.item = item
orig_sync = torch.cuda.Stream.synchronize
def ssync(self):
    t = time.perf_counter(); r = orig_sync(self); log.append(("ssync", "", t - t0[0], time.perf_counter() - t)); return r
torch.cuda.Stream.synchronize = ssync
orig_cpu = torch.Tensor.cpu
def cpu(self, *a, **k):
    t = time.perf_counter(); r = orig_cpu(self, *a, **k); log.append(("cpu", str(tuple(self.shape)), t - t0[0], time.perf_counter() - t)); return r
torch.Tensor.cpu = cpu
for it in range(3):
    m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    torch.cuda.synchronize()
    log.clear()
    t0[0] = time.perf_counter()
    res, rep = sx.run_pipeline(m, k=w.k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters, seed=w.seed)
    _ = res.item_ids
    torch.cuda.synchronize()
    total = time.perf_counter() - t0[0]
for kind, name, ts, dur in log:
    if dur > 2e-4 or kind != "call":
        print(f"{ts*1e3:8.2f} ms  {kind:5s} {name:28s} {dur*1e3:7.3f} ms")
print("total", total * 1e3, "ms; calls", sum(1 for l in log if l[0] == "call"))
