import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1706_01449_b200 as sx
rng = np.random.default_rng(0)
u = rng.normal(size=(3000, 20))
cl = sx.kmeans(sx.FactorMatrix(u), 16, max_iters=5, seed=1)
print("ok", cl.assignment[:10])
