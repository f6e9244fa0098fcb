import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "oracle"))
import numpy as np, torch
import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _ops
rng = np.random.default_rng(3)
base = rng.normal(size=(4, 6))
users = base[rng.integers(0, 4, 500)]
r2 = np.random.default_rng(2)
first = int(r2.integers(0, 500)); unif = r2.random(5)
p = torch.as_tensor(users, device="cuda")
rows, cen, deg = _ops.kmeans_seed(p, 6, first, torch.as_tensor(unif, device="cuda"))
print("gpu rows", rows.cpu().numpy(), "deg", int(deg.item()))
import os as _o
_o.environ["SIMDEX_SEED_NO_F16"] = "1"
rows, cen, deg = _ops.kmeans_seed(p, 6, first, torch.as_tensor(unif, device="cuda"))
print("gpu rows nof16", rows.cpu().numpy(), "deg", int(deg.item()))
