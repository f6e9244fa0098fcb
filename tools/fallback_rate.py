"""Exact-fallback rows of the brute-force pass on log-normal(0, sigma) user
norms, one matrix-wide fp16 scale vs one scale per row.
    python tools/fallback_rate.py [sigma]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _device, _lib, _ops

sigma = float(sys.argv[1]) if len(sys.argv) > 1 else 3.0
rng = np.random.default_rng(17)
nu, ni, f, k = 200_000, 17_770, 50, 10
users = (rng.normal(size=(nu, f)) * rng.lognormal(0.0, sigma, (nu, 1))).astype(np.float32).astype(np.float64)
items = (rng.normal(size=(ni, f)) * rng.lognormal(0.0, 0.5, (ni, 1))).astype(np.float32).astype(np.float64)
m = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
u, it = _device.f64(m.users), _device.f64(m.items)
pi = _device.packed_sorted(m.items)
for name, pu in (("matrix-wide scale", _device.packed(m.users)), ("per-row scale", _device.packed_users(m.users))):
    for _ in range(2):
        _ops.topk_matmul(u, pu, it, pi, k, items32=_device.f32_exact(m.items), users32=_device.f32_exact(m.users))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ids, sc, _ = _ops.topk_matmul(u, pu, it, pi, k, items32=_device.f32_exact(m.items),
                                  users32=_device.f32_exact(m.users))
    e1.record()
    torch.cuda.synchronize()
    print(f"sigma={sigma} {name:18s}: fallback rows {_lib.fallback_rows():7d} of {nu} "
          f"({_lib.fallback_rows() / nu:.3%}), {e0.elapsed_time(e1):.2f} ms")
