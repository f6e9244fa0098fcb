"""CUDA-event time of the k-means++ seeding alone (no timers inside the
kernel): python tools/time_seed.py [cfg] [reps]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import _device, _ops
from paper_1706_01449_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = W.CONFIGS[cfg]()
users = sx.FactorMatrix(w.users)
pts = _device.f64(users)
p32 = _device.f32_exact(users)
rng = np.random.default_rng(w.seed)
first = int(rng.integers(0, users.rows))
unif = _device.to_device(rng.random(w.clusters - 1))
times = []
for r in range(reps + 1):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    rows, cen, deg = _ops.kmeans_seed(pts, w.clusters, first, unif, points32=p32)
    b.record()
    torch.cuda.synchronize()
    if r:
        times.append(a.elapsed_time(b))
print(f"{cfg} seeding {w.clusters} seeds over {users.rows} points: median {np.median(times):.3f} ms "
      f"(min {min(times):.3f}); rows checksum {int(rows.sum().item())}")
