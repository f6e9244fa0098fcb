"""How much catalogue-pass work a list-order stage 2 would do: per cluster,
continuing users (no-WS walk w_u > B') in 32-row warps; a warp runs until its
longest walk (Algorithm 1's stop on the list ceilings), in 128-item tiles.
Compares with the norm-sorted pass's executed pairs.  python tools/stage2_list_potential.py [cfg] [k]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _lib, optimizer
from paper_1706_01449_b200 import index as I
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
plan = optimizer.plan_pipeline(m, k=k, num_clusters=w.clusters, block_size=4096, max_iters=w.max_iters, seed=w.seed)
idx = plan.index
n = m.num_items
B = min(4096, n)
_, _, vis = I.query_batch_tensors(idx, m, None, k, work_sharing=False)
wu = vis.cpu().numpy()
I.query_batch_tensors(idx, m, None, k, work_sharing=True)
torch.cuda.synchronize()
p1, p2 = _lib.executed_pairs()
a = np.asarray(idx.clustering.assignment)
cont = wu > B
print(f"{cfg} k={k}: continuing users {cont.sum()} of {wu.size}; mean w_u of them {wu[cont].mean():.0f}; "
      f"norm-sorted pass executed {p2} pairs = {p2 / max(cont.sum(), 1):.0f} per continuing user")
tiles = 0
rows_tiles = 0
for c in range(idx.num_clusters):
    sel = np.sort(wu[(a == c) & cont] - B)  # walks past B' of this cluster's continuing users (packed by cluster)
    # the packed order is by user id within the cluster; use that order
    ids = np.flatnonzero((a == c) & cont)
    ext = wu[ids] - B
    for s in range(0, ext.size, 32):
        mx = ext[s:s + 32].max()
        tiles += int(np.ceil(mx / 128))
    rows_tiles += int(np.ceil(ext / 128).sum()) if ext.size else 0
print(f"  list order: warp-tiles {tiles} (x 32 rows x 128 items = {tiles * 32 * 128} pairs); "
      f"per-row tiles {rows_tiles} ({rows_tiles * 128} pairs)")
