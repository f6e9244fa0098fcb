import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _device, _ops, index as I
spec = sx.SyntheticSpec(200, 500, 8, archetype_count=6, angular_spread=0.5, norm_low=0.5, norm_high=2.5, seed=42)
m = sx.generate_synthetic(spec)
cl = sx.kmeans(m.users, 6, seed=1)
idx = sx.build_index(m, cl, 64)
k = 7
want = sx.topk_naive(m, k)
u = _device.f64(m.users)
pm = _device.packed(m.users)
pr = _ops.pack_rows(u)
print("matrix su", pm.scale_exp, "row exps", np.unique(pr.row_exp.cpu().numpy(), return_counts=True))
variants = {
    "matrix": pm,
    "rows": pr,
    "matrix-op+const-exp": _ops.Packed(pm.op, pm.norms, 0, pm.kp, pm.rows, row_exp=torch.full_like(pr.row_exp, pm.scale_exp)),
    "rows-op-compare": None,
}
print("op equal where exp==su:", end=" ")
re = pr.row_exp.cpu().numpy()
sel = np.flatnonzero(re == pm.scale_exp)
print(bool((pm.op[sel] == pr.op[sel]).all().item()), len(sel))
pi = _device.packed_sorted(m.items)
ids, bounds = idx.device_lists()
grouped = _ops.group_queries(torch.arange(200, device=u.device), idx.device_assignment(), idx.num_clusters)
for name, pu in variants.items():
    if pu is None:
        continue
    out = _ops.query_ws(u, pu, _device.f64(m.items), pi, ids, idx.device_list_pos(), bounds, 64, idx.device_prefix(m), grouped, k,
                        items32=_device.f32_exact(m.items), users32=_device.f32_exact(m.users))
    got = out[0].cpu().numpy()
    bad = np.flatnonzero((got != want.item_ids).any(axis=1))
    print(name, "bad", bad[:8], len(bad))
    out = _ops.topk_matmul(u, pu, _device.f64(m.items), pi, k, items32=_device.f32_exact(m.items), users32=_device.f32_exact(m.users))
    got = out[0].cpu().numpy()
    bad = np.flatnonzero((got != want.item_ids).any(axis=1))
    print(name, "brute bad", bad[:8], len(bad))
