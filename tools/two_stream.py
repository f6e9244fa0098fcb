"""Prototype: a rank's serving step as P concurrent work-sharing calls (its
users cut into P cluster-ordered parts, one execution context and one stream
each, fork/join by events), eager and graph-replayed, against the single
call.  python tools/two_stream.py [cfg] [N] [rank] [P]"""
import ctypes as C
import os
import statistics
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _lib, graphs, index as I, optimizer, sharding
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
r = int(sys.argv[3]) if len(sys.argv) > 3 else 0
P = int(sys.argv[4]) if len(sys.argv) > 4 else 2
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
plan = optimizer.plan_pipeline(m, k=w.k, num_clusters=w.clusters or 8, block_size=4096, max_iters=w.max_iters,
                               seed=w.seed)
idx = plan.index
if n == 1:
    uids = np.arange(m.num_users)
else:
    uids = sharding.IndexShard(idx, m, r, n, plan.walk).user_ids
asg = np.asarray(idx.clustering.assignment)[uids]
order = np.argsort(asg, kind="stable")
parts = [I.QuerySet(idx, np.sort(uids[order[len(order) * i // P: len(order) * (i + 1) // P]])) for i in range(P)]
whole = I.QuerySet(idx, uids)
lib = _lib.load()
ctxs = []
for _ in range(P):
    h = C.c_void_p()
    _lib.call("simdex_ctx_create", 0, C.byref(h))
    ctxs.append(h)
streams = [torch.cuda.Stream() for _ in range(P)]
flush = torch.empty(256 << 20, dtype=torch.int8, device="cuda")


def single():
    return I.query_batch_tensors(idx, m, whole, w.k)


def multi():
    main = torch.cuda.current_stream()
    ev0 = torch.cuda.Event()
    ev0.record(main)
    outs = []
    for q, c, st in zip(parts, ctxs, streams):
        st.wait_event(ev0)
        with torch.cuda.stream(st):
            outs.append(I.query_batch_tensors(idx, m, q, w.k, ctx=c))
    for st in streams:
        e = torch.cuda.Event()
        e.record(st)
        main.wait_event(e)
    return outs


def timed(fn, steps=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for s in range(steps):
        flush.fill_(s & 0x7F)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


res = {"cfg": cfg, "n": n, "rank": r, "P": P, "users": int(uids.size)}
res["single_eager"] = timed(single)
res["multi_eager"] = timed(multi)
res["single_graph"] = timed(graphs.GraphedCall(single))
res["multi_graph"] = timed(graphs.GraphedCall(lambda: tuple(x for o in multi() for x in o)))
# correctness: same rows
a = single()
b = multi()
ida = a[0].cpu().numpy()
pos = {u: i for i, u in enumerate(whole.user_ids)}
ok = all(np.array_equal(ida[[pos[u] for u in q.user_ids]], o[0].cpu().numpy()) for q, o in zip(parts, b))
res["ids_equal"] = bool(ok)
print(res)
