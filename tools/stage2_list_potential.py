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

# stage 1 (the prefix): with list order and a per-warp stop on the ceilings,
# a warp of 32 consecutive packed rows of a cluster needs min(B', its longest
# walk) items; the prefix pass multiplies B' for every row
tiles1 = 0
full1 = 0
for c in range(idx.num_clusters):
    ids = np.flatnonzero(a == c)
    ext = np.minimum(wu[ids], B)
    for s in range(0, ext.size, 32):
        tiles1 += int(np.ceil(ext[s:s + 32].max() / 128))
        full1 += B // 128
print(f"  stage 1: per-warp stop on the ceilings needs {tiles1} warp-tiles of {full1} ({tiles1 / full1:.2f})")
for grp in (32, 128):
    for sort in (False, True):
        t = 0
        for c in range(idx.num_clusters):
            ext = np.minimum(wu[np.flatnonzero(a == c)], B)
            if sort:
                ext = np.sort(ext)
            for s in range(0, ext.size, grp):
                t += int(np.ceil(ext[s:s + grp].max() / 128)) * (grp // 32)
        print(f"  stage 1, groups of {grp} rows {'sorted by walk' if sort else 'packed order'}: {t / full1:.2f} of the warp-tiles")
# a cheap proxy for the walk: the user's angle to its centroid
cen = np.asarray(idx.clustering.centroids.values)
U = m.users.values
cosv = np.einsum('ij,ij->i', U, cen[a]) / (np.linalg.norm(U, axis=1) * np.linalg.norm(cen[a], axis=1) + 1e-300)
t = 0
for c in range(idx.num_clusters):
    ids = np.flatnonzero(a == c)
    ext = np.minimum(wu[ids], B)[np.argsort(-cosv[ids])]
    for s in range(0, ext.size, 128):
        t += int(np.ceil(ext[s:s + 128].max() / 128)) * 4
print(f"  stage 1, units of 128 sorted by angle to the centroid: {t / full1:.2f}")
