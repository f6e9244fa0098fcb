import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _device
spec = sx.SyntheticSpec(200, 500, 8, archetype_count=6, angular_spread=0.5, norm_low=0.5, norm_high=2.5, seed=42)
m = sx.generate_synthetic(spec)
cl = sx.kmeans(m.users, 6, seed=1)
idx = sx.build_index(m, cl, 64)
for k in (1, 7, 50):
    want = sx.topk_naive(m, k)
    for ws in (True, False):
        got = sx.query_batch(idx, m, None, k, work_sharing=ws)
        bad = np.flatnonzero((got.item_ids != want.item_ids).any(axis=1))
        print("k", k, "ws", ws, "bad", bad[:10], len(bad))
        if len(bad):
            pu = _device.packed_users(m.users)
            re = pu.row_exp.cpu().numpy() if pu.row_exp is not None else None
            for u in bad[:3]:
                print("  user", u, "norm", np.linalg.norm(m.users.values[u]), "exp", None if re is None else re[u],
                      "got", got.item_ids[u][:5], got.visited[u], "want", want.item_ids[u][:5])
