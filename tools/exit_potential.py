"""How much of the stage-1 prefix a ceiling-based early exit could skip:
per-user Algorithm 1 stop positions (query_batch without work sharing gives
visited = the stop position) grouped into 128-user units in the serving
order (by cluster, user id) vs sorted by a difficulty proxy / by the stop
itself.  python tools/exit_potential.py [cfg] [k]"""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W, index as I
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
k = int(sys.argv[2]) if len(sys.argv) > 2 else 10
w = W.CONFIGS[cfg]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
cl = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
idx = sx.build_index(m, cl, 4096)
ids, sc, vis = I.query_batch_tensors(idx, m, None, k, False)
vis = vis.cpu().numpy()
B = min(4096, m.num_items)
stop_t = np.ceil(np.minimum(vis, B) / 128.0)
lab = np.asarray(cl.assignment)
full = 0; used = {"serving order": 0, "cos to centroid": 0, "user norm": 0, "oracle": 0}
U = m.users.values; cen = np.asarray(cl.centroids.values)
for c in range(cl.num_clusters if hasattr(cl, "num_clusters") else cen.shape[0]):
    mem = np.flatnonzero(lab == c)
    if mem.size == 0:
        continue
    x = U[mem]; un = np.linalg.norm(x, axis=1)
    cosu = x @ cen[c] / (un * np.linalg.norm(cen[c]) + 1e-300)
    orders = {"serving order": np.arange(mem.size), "cos to centroid": np.argsort(-cosu, kind="stable"),
              "user norm": np.argsort(un, kind="stable"), "oracle": np.argsort(stop_t[mem], kind="stable")}
    nun = -(-mem.size // 128)
    full += nun * (B / 128.0)
    for name, o in orders.items():
        st = stop_t[mem][o]
        pad = np.zeros(nun * 128); pad[:st.size] = st
        used[name] += pad.reshape(nun, 128).max(axis=1).sum()
print(f"{cfg} K={k}: users continuing past B {np.mean(vis > B):.3f}, mean stop {vis.mean():.0f}")
for name, v in used.items():
    print(f"  {name:16s} tiles needed {v / full:.3f} of the prefix")
