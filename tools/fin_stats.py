"""Candidate-buffer and survivor counts per finalize mode for one serving call
(diagnostic build: make EXTRA=-DSIMDEX_FIN_STATS=1 OBJDIR=../../build/ab/objS
LIB=../../build/ab/libS.so, then SIMDEX_LIB_PATH=build/ab/libS.so
python tools/fin_stats.py cfg2 10)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _lib, optimizer
from paper_1706_01449_b200 import index as index_mod
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
ks = [int(x) for x in sys.argv[2:]] or [10]
w = W.CONFIGS[cfg]()
model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
lib = _lib.load()
fn = lib.simdex_dbg_fin_stats
buf = (C.c_ulonglong * 12)()
if cfg in ("cfg1", "cfg3", "cfg5"):
    plan = None
else:
    plan = optimizer.plan_pipeline(model, k=ks[0], num_clusters=w.clusters, block_size=4096,
                                   max_iters=w.max_iters, seed=w.seed)
for k in ks:
    if plan is None:
        step = lambda: sx.brute.topk_matmul_tensors(model, k)  # noqa: E731
    else:
        step = lambda: index_mod.query_batch_tensors(plan.index, model, None, k)  # noqa: E731
    step()
    torch.cuda.synchronize()
    fn(buf)
    step()
    torch.cuda.synchronize()
    fn(buf)
    for mode, name in ((0, "brute"), (1, "prefix"), (2, "full-list"), (3, "assign")):
        cnt, kept, rows = buf[3 * mode], buf[3 * mode + 1], buf[3 * mode + 2]
        if rows:
            print(f"{cfg} k={k} {name}: rows {rows}, buffered {cnt / rows:.1f} per row, survivors {kept / rows:.1f} per row")
