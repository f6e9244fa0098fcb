"""Generate golden vectors from the REFERENCE package (run in the build
container, where /root/reference exists).  TEST INFRASTRUCTURE ONLY.

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py [--big]

Imports ``mipserve`` from /root/reference/pkg/src (read-only) and writes
``tests/golden/*.npz``: inputs plus the reference's own outputs for the hot
path (topk_naive / topk_matmul / kmeans / compute_max_angles / build_index /
query_user / query_batch / estimate_walk_length / decide).  These fixtures
pin both ``oracle/simdex_oracle.py`` (CPU tests) and the CUDA path (GPU
tests); nothing at test time reads /root/reference.

``--big`` adds the BASELINE cfg1 full-size brute-force answers and the cfg2
full-size clustering/index/walk-sample answers (slow: the reference's
k-means at cfg2 takes ~1 minute).  ``--cfg2-k5`` adds K = 5 to the cfg2
fixture (same clustering, which the fixture stores).  ``--cfg4 FILE``
writes the cfg4 fixture from a GPU clustering dumped on the box
(tools/dump_clustering.py): the reference's compute_max_angles,
build_index, query_batch and query_user on that clustering for a 500-user
sample.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import mipserve as M  # noqa: E402  (the reference)
from mipserve import optimizer as MO  # noqa: E402


def spec_model(nu, ni, f, archetypes=8, spread=0.3, norms=(0.5, 2.5), seed=0):
    """Same helper shape as the reference's tests/conftest.py make_model."""
    spec = M.SyntheticSpec(nu, ni, f, archetype_count=min(archetypes, nu), angular_spread=spread,
                           norm_low=norms[0], norm_high=norms[1], seed=seed)
    return M.generate_synthetic(spec)


def arr(results, attr):
    return np.stack([getattr(r, attr) for r in results])


def small_cases():
    cases = []
    rng = np.random.default_rng(20260808)
    # (users, items, f, archetypes, spread, norms, seed)
    shapes = [
        (50, 140, 6, 8, 0.3, (0.3, 3.0), 3),
        (200, 500, 8, 6, 0.5, (0.5, 2.5), 42),
        (120, 1000, 25, 10, 0.4, (0.5, 2.5), 12),
        (60, 150, 5, 60, 0.0, (0.5, 2.5), 9),
        (300, 700, 50, 16, 0.6, (0.5, 2.5), 77),
        (40, 60, 2, 4, 0.9, (0.5, 5.0), 5),
        (25, 33, 1, 2, 0.0, (0.5, 2.0), 6),
        (600, 2500, 16, 8, 0.03, (1.0, 1.1), 31),
    ]
    for i, (nu, ni, f, a, s, nr, seed) in enumerate(shapes):
        cases.append((f"syn{i}", spec_model(nu, ni, f, a, s, nr, seed)))
    # exact score ties: duplicated item rows (reference tests/test_brute.py:63-71)
    base = np.random.default_rng(9).normal(size=(12, 5))
    cases.append(("dups", M.ModelPair(M.FactorMatrix(np.random.default_rng(10).normal(size=(9, 5))),
                                     M.FactorMatrix(np.vstack([base, base[:6]])))))
    # zero-norm user and zero-norm item (tests/test_index.py:107-115, :150-157)
    u = np.vstack([np.zeros(4), np.ones(4), rng.normal(size=(6, 4))])
    it = np.vstack([rng.normal(size=(20, 4)), np.zeros((1, 4)), rng.normal(size=(9, 4))])
    cases.append(("zeros", M.ModelPair(M.FactorMatrix(u), M.FactorMatrix(it))))
    # integer-valued data with many exact ties
    ui = rng.integers(-2, 3, size=(30, 3)).astype(float)
    ii = rng.integers(-2, 3, size=(40, 3)).astype(float)
    cases.append(("intties", M.ModelPair(M.FactorMatrix(ui), M.FactorMatrix(ii))))
    return cases


def dump_case(name, model, ks=(1, 5, 10, 50), clusters=(1, 4), blocks=(4096, 64, 1)):
    t0 = time.time()
    users, items = model.users.values, model.items.values
    out = {"users": users, "items": items, "ks": np.array(ks)}
    n = model.num_items
    for k in ks:
        nv = M.topk_naive(model, k)
        out[f"naive_ids_k{k}"] = arr(nv, "item_ids")
        out[f"naive_scores_k{k}"] = arr(nv, "scores")
        cnt = {}
        mm = M.topk_matmul(model, k, counters=cnt)
        out[f"matmul_ids_k{k}"] = arr(mm, "item_ids")
        out[f"heap_ops_k{k}"] = cnt["heap_ops"]
    out["clusters"] = np.array([c for c in clusters if c <= model.num_users])
    for c in out["clusters"]:
        cl = M.kmeans(model.users, int(c), max_iters=100, seed=int(c) + 1)
        out[f"km{c}_centroids"] = cl.centroids.values
        out[f"km{c}_assignment"] = cl.assignment
        out[f"km{c}_max_angle"] = cl.max_angle
        out[f"km{c}_objective"] = cl.objective
        for b in blocks:
            idx = M.build_index(model, cl, b)
            if b == blocks[0]:
                out[f"km{c}_list_ids"] = idx.item_ids
                out[f"km{c}_bounds"] = idx.bounds
                out[f"km{c}_item_norms"] = idx.item_norms
            for k in ks:
                if b == blocks[0]:
                    qu = [M.query_user(idx, model, u, k) for u in range(model.num_users)]
                    out[f"km{c}_k{k}_user_ids"] = arr(qu, "item_ids")
                    out[f"km{c}_k{k}_user_scores"] = arr(qu, "scores")
                    out[f"km{c}_k{k}_user_visited"] = np.array([r.visited for r in qu])
                ws = M.query_batch(idx, model, None, k, work_sharing=True)
                out[f"km{c}_b{b}_k{k}_ws_ids"] = arr(ws, "item_ids")
                out[f"km{c}_b{b}_k{k}_ws_visited"] = np.array([r.visited for r in ws])
            est = MO.estimate_walk_length(idx, model, 0.05, ks[-1 if len(ks) < 3 else 2], seed=int(c))
            out[f"km{c}_est"] = np.array([est.mean_visited, est.ci_low, est.ci_high, est.sample_size])
            out[f"km{c}_est_ids"] = np.array(sorted(est.sampled))
    out["blocks"] = np.array(blocks)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    print(f"{name}: {model.num_users}x{n}x{model.factors} in {time.time() - t0:.1f}s", flush=True)


def decisions():
    # the 64 Table-2 cells (reference tests/test_acceptance.py:198-233)
    fr = [
        [0.032, 0.058, 0.092, 0.176], [0.375, 0.477, 0.542, 0.700], [0.699, 0.786, 0.842, 0.898],
        [0.135, 0.210, 0.241, 0.339], [0.039, 0.109, 0.112, 0.231], [0.358, 0.440, 0.515, 0.676],
        [0.570, 0.668, 0.712, 0.817], [0.576, 0.651, 0.697, 0.827], [0.022, 0.036, 0.044, 0.069],
        [0.050, 0.063, 0.074, 0.104], [0.0317, 0.038, 0.043, 0.067], [0.0, 0.0, 0.0, 0.0],
        [0.0482, 0.092, 0.117, 0.168], [0.271, 0.358, 0.403, 0.500], [0.503, 0.597, 0.618, 0.691],
        [0.552, 0.623, 0.649, 0.716],
    ]
    n = 1 << 20
    got = [[M.decide(f * n, n, 0, k, 0.05) for f, k in zip(row, (1, 5, 10, 50))] for row in fr]
    hf = [M.hardware_factor(k, 0.05) for k in (1, 2, 5, 10, 50, 500)]
    np.savez_compressed(os.path.join(OUT, "decisions.npz"), fractions=np.array(fr),
                        picks=np.array(got), hw_factor=np.array(hf))


def big():
    from paper_1706_01449_b200 import workloads as W
    t0 = time.time()
    w = W.cfg1()
    model = M.ModelPair(M.FactorMatrix(w.users), M.FactorMatrix(w.items))
    nv = M.topk_naive(model, 10)
    np.savez_compressed(os.path.join(OUT, "cfg1_k10.npz"), ids=arr(nv, "item_ids").astype(np.int16),
                        scores=arr(nv, "scores"))
    print(f"cfg1 naive in {time.time() - t0:.1f}s", flush=True)

    t0 = time.time()
    w = W.cfg2()
    model = M.ModelPair(M.FactorMatrix(w.users), M.FactorMatrix(w.items))
    cl = M.kmeans(model.users, 256, max_iters=3, seed=1)
    print(f"cfg2 kmeans in {time.time() - t0:.1f}s", flush=True)
    idx = M.build_index(model, cl, 4096)
    rng = np.random.default_rng(123)
    sample = np.sort(rng.choice(model.num_users, 2000, replace=False))
    out = {"centroids": cl.centroids.values, "assignment": cl.assignment.astype(np.int16),
           "max_angle": cl.max_angle, "objective": cl.objective, "sample": sample,
           "bounds_head": idx.bounds[:, :64], "ids_head": idx.item_ids[:, :64].astype(np.int16)}
    for k in (1, 10, 50):
        est = MO.estimate_walk_length(idx, model, 0.001, k, seed=1)
        out[f"est_k{k}"] = np.array([est.mean_visited, est.ci_low, est.ci_high, est.sample_size])
        ws = M.query_batch(idx, model, sample, k, work_sharing=True)
        out[f"ws_k{k}_ids"] = arr(ws, "item_ids").astype(np.int16)
        out[f"ws_k{k}_scores"] = arr(ws, "scores")
        out[f"ws_k{k}_visited"] = np.array([r.visited for r in ws], dtype=np.int32)
        nows = [M.query_user(idx, model, int(u), k) for u in sample[:500]]
        out[f"nows_k{k}_visited"] = np.array([r.visited for r in nows], dtype=np.int32)
    np.savez_compressed(os.path.join(OUT, "cfg2_index.npz"), **out)
    print(f"cfg2 golden in {time.time() - t0:.1f}s", flush=True)


def _ref_clustering(cen, assign, seed, users):
    c = cen.shape[0]
    theta = M.compute_max_angles(users, M.FactorMatrix(cen), assign)
    return M.Clustering(M.FactorMatrix(cen), assign, theta, tuple(np.flatnonzero(assign == j) for j in range(c)),
                        np.empty(0), seed)


def cfg2_k5():
    """K = 5 (a BASELINE depth) on the stored cfg2 reference clustering."""
    from paper_1706_01449_b200 import workloads as W
    t0 = time.time()
    path = os.path.join(OUT, "cfg2_index.npz")
    g = dict(np.load(path))
    w = W.cfg2()
    model = M.ModelPair(M.FactorMatrix(w.users), M.FactorMatrix(w.items))
    cl = _ref_clustering(g["centroids"], g["assignment"].astype(np.int64), 1, model.users)
    np.testing.assert_array_equal(cl.max_angle, g["max_angle"])  # the stored clustering is the reference's
    idx = M.build_index(model, cl, 4096)
    sample = g["sample"]
    k = 5
    est = MO.estimate_walk_length(idx, model, 0.001, k, seed=1)
    g[f"est_k{k}"] = np.array([est.mean_visited, est.ci_low, est.ci_high, est.sample_size])
    ws = M.query_batch(idx, model, sample, k, work_sharing=True)
    g[f"ws_k{k}_ids"] = arr(ws, "item_ids").astype(np.int16)
    g[f"ws_k{k}_scores"] = arr(ws, "scores")
    g[f"ws_k{k}_visited"] = np.array([r.visited for r in ws], dtype=np.int32)
    nows = [M.query_user(idx, model, int(u), k) for u in sample[:500]]
    g[f"nows_k{k}_visited"] = np.array([r.visited for r in nows], dtype=np.int32)
    np.savez_compressed(path, **g)
    print(f"cfg2 K=5 in {time.time() - t0:.1f}s", flush=True)


def cfg4_fixture(dump_path):
    """cfg4 (1,823,179 x 136,736, C=1024) answers of the reference on the GPU
    clustering: only the sampled users' clusters are built (a cluster's list
    depends on its centroid and theta_b alone, index.py:129-155)."""
    from paper_1706_01449_b200 import workloads as W
    t0 = time.time()
    d = np.load(dump_path)
    cen, assign = d["centroids"], d["assignment"].astype(np.int64)
    w = W.cfg4()
    users = M.FactorMatrix(w.users)
    items = M.FactorMatrix(w.items)
    theta_all = M.compute_max_angles(users, M.FactorMatrix(cen), assign)
    rng = np.random.default_rng(404)
    clusters = np.sort(rng.choice(np.unique(assign), 40, replace=False))
    pool = np.flatnonzero(np.isin(assign, clusters))
    sample = np.sort(rng.choice(pool, 500, replace=False))
    # the reference index over the chosen clusters only (same lists, fewer of them)
    remap = {int(c): j for j, c in enumerate(clusters)}
    sub_assign = np.array([remap.get(int(a), 0) for a in assign[sample]], dtype=np.int64)
    sub_users = M.FactorMatrix(w.users[sample])
    sub_model = M.ModelPair(sub_users, items)
    sub_cl = M.Clustering(M.FactorMatrix(cen[clusters]), sub_assign, theta_all[clusters],
                          tuple(np.flatnonzero(sub_assign == j) for j in range(clusters.size)), np.empty(0), 3)
    idx = M.build_index(sub_model, sub_cl, 4096)
    out = {"centroids": cen, "assignment_sha": np.frombuffer(__import__("hashlib").sha256(
        assign.astype("<i8").tobytes()).digest(), dtype=np.uint8), "theta": theta_all, "sample": sample,
        "clusters": clusters}
    for k in (1, 10):
        ws = M.query_batch(idx, sub_model, None, k, work_sharing=True)
        out[f"ws_k{k}_ids"] = arr(ws, "item_ids").astype(np.int32)
        out[f"ws_k{k}_scores"] = arr(ws, "scores")
        out[f"ws_k{k}_visited"] = np.array([r.visited for r in ws], dtype=np.int32)
        nows = [M.query_user(idx, sub_model, i, k) for i in range(sample.size)]
        out[f"nows_k{k}_ids"] = arr(nows, "item_ids").astype(np.int32)
        out[f"nows_k{k}_visited"] = np.array([r.visited for r in nows], dtype=np.int32)
    np.savez_compressed(os.path.join(OUT, "cfg4_sample.npz"), **out)
    print(f"cfg4 fixture in {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    if "--cfg2-k5" in sys.argv:
        cfg2_k5()
        sys.exit(0)
    if "--cfg4" in sys.argv:
        cfg4_fixture(sys.argv[sys.argv.index("--cfg4") + 1])
        sys.exit(0)
    os.makedirs(OUT, exist_ok=True)
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    decisions()
    for name, model in small_cases():
        dump_case(name, model)
    if "--big" in sys.argv:
        big()
