"""Dump the GPU k-means clustering of a BASELINE config (for
oracle/make_golden.py --cfg4, which runs the reference on it):
    python tools/dump_clustering.py --config cfg4 --out gpurun_out/cfg4_gpu_clustering.npz"""
import argparse
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np

import paper_1706_01449_b200 as sx
from paper_1706_01449_b200 import workloads as W

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--out", required=True)
a = ap.parse_args()
w = W.CONFIGS[a.config]()
m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
cl = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)
a2 = sx.kmeans(m.users, w.clusters, max_iters=w.max_iters, seed=w.seed)  # determinism check
same = np.array_equal(cl.centroids.values, a2.centroids.values) and np.array_equal(cl.assignment, a2.assignment)
np.savez_compressed(a.out, centroids=cl.centroids.values, assignment=np.asarray(cl.assignment).astype(np.int16),
                    max_angle=cl.max_angle)
print("dumped", a.out, "deterministic", same)
