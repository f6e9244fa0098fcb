"""GPU parity: every hot-path function of the package against the reference's
own outputs (tests/golden, generated from mipserve) and the CPU oracle.
Ids must match exactly; scores within rtol=atol=1e-9 (the reference's own
tolerance, tests/conftest.py:41-47)."""

import numpy as np
import pytest

from conftest import assert_lists_equal_up_to_ties, assert_same_topk, canonical_ids, golden_names, load_golden

pytestmark = pytest.mark.gpu

NAMES = golden_names()


@pytest.fixture(scope="module")
def sx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_01449_b200 as pkg
    return pkg


def _model(sx, g):
    return sx.ModelPair(sx.FactorMatrix(g["users"]), sx.FactorMatrix(g["items"]))


def _ids(res):
    return np.stack([r.item_ids for r in res])


def _scores(res):
    return np.stack([r.scores for r in res])


def _ref_clustering(sx, g, c):
    a = g[f"km{c}_assignment"]
    return sx.Clustering(sx.FactorMatrix(g[f"km{c}_centroids"]), a, g[f"km{c}_max_angle"],
                         tuple(np.flatnonzero(a == j) for j in range(int(c))), g[f"km{c}_objective"], int(c) + 1)


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("path", ["naive", "matmul"])
def test_brute_force_matches_reference(sx, name, path):
    g = load_golden(name)
    model = _model(sx, g)
    fn = sx.topk_naive if path == "naive" else sx.topk_matmul
    for k in g["ks"]:
        res = fn(model, int(k))
        assert len(res) == model.num_users
        if name == "dups":
            np.testing.assert_array_equal(canonical_ids(g["items"], _ids(res)),
                                          canonical_ids(g["items"], g[f"naive_ids_k{k}"]))
            np.testing.assert_allclose(_scores(res), g[f"naive_scores_k{k}"], rtol=1e-9, atol=1e-9)
        else:
            assert_same_topk(_ids(res), _scores(res), g[f"naive_ids_k{k}"], g[f"naive_scores_k{k}"],
                             ctx=f"{name} {path} k={k}")


@pytest.mark.parametrize("name", NAMES)
def test_kmeans_matches_reference(sx, name):
    g = load_golden(name)
    model = _model(sx, g)
    for c in g["clusters"]:
        cl = sx.kmeans(model.users, int(c), max_iters=100, seed=int(c) + 1)
        np.testing.assert_array_equal(cl.assignment, g[f"km{c}_assignment"])
        # in-order member sums: bit-identical to the reference's numpy means
        np.testing.assert_array_equal(cl.centroids.values, g[f"km{c}_centroids"])
        np.testing.assert_allclose(cl.max_angle, g[f"km{c}_max_angle"], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(cl.objective, g[f"km{c}_objective"], rtol=1e-12, atol=1e-12)
        assert sorted(np.concatenate(cl.members).tolist()) == list(range(model.num_users))
        for j, ms in enumerate(cl.members):
            assert ms.size > 0 and np.all(cl.assignment[ms] == j)


@pytest.mark.parametrize("name", NAMES)
def test_build_index_matches_reference(sx, name):
    g = load_golden(name)
    model = _model(sx, g)
    for c in g["clusters"]:
        idx = sx.build_index(model, _ref_clustering(sx, g, c), 64)
        if name == "intties":  # integer data: exact mathematical ties in the ceilings
            assert_lists_equal_up_to_ties(idx.item_ids, idx.bounds, g[f"km{c}_list_ids"], g[f"km{c}_bounds"])
        else:
            np.testing.assert_array_equal(idx.item_ids, g[f"km{c}_list_ids"])
            np.testing.assert_allclose(idx.bounds, g[f"km{c}_bounds"], rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(idx.item_norms, g[f"km{c}_item_norms"], rtol=1e-14)
        assert idx.entry_count == int(c) * model.num_items
        assert all(np.all(np.diff(idx.bounds[j]) <= 0.0) for j in range(int(c)))


@pytest.mark.parametrize("name", NAMES)
def test_walks_match_reference(sx, name):
    g = load_golden(name)
    model = _model(sx, g)
    for c in g["clusters"]:
        cl = _ref_clustering(sx, g, c)
        for b in g["blocks"]:
            idx = sx.build_index(model, cl, int(b))
            for k in g["ks"]:
                k = int(k)
                if b == g["blocks"][0]:
                    off = sx.query_batch(idx, model, None, k, work_sharing=False)
                    ctx = f"{name} C={c} k={k}"
                    if name == "dups":
                        np.testing.assert_array_equal(canonical_ids(g["items"], _ids(off)),
                                                      canonical_ids(g["items"], g[f"km{c}_k{k}_user_ids"]))
                    else:
                        assert_same_topk(_ids(off), _scores(off), g[f"km{c}_k{k}_user_ids"],
                                         g[f"km{c}_k{k}_user_scores"], ctx=ctx)
                    if name == "intties":
                        # integer data: kth == ceiling*||u|| exactly in real arithmetic for some
                        # positions, so the strict stop test is decided by last-ulp rounding
                        continue
                    np.testing.assert_array_equal(off.visited, g[f"km{c}_k{k}_user_visited"], err_msg=ctx)
                    u = model.num_users // 2
                    one = sx.query_user(idx, model, u, k)
                    assert one.visited == g[f"km{c}_k{k}_user_visited"][u]
                ws = sx.query_batch(idx, model, None, k, work_sharing=True)
                if name != "dups":
                    np.testing.assert_array_equal(_ids(ws), g[f"km{c}_b{b}_k{k}_ws_ids"])
                if name != "intties":
                    np.testing.assert_array_equal(ws.visited, g[f"km{c}_b{b}_k{k}_ws_visited"])


@pytest.mark.parametrize("name", NAMES)
def test_walk_estimate_matches_reference(sx, name):
    g = load_golden(name)
    model = _model(sx, g)
    for c in g["clusters"]:
        idx = sx.build_index(model, _ref_clustering(sx, g, c), 4096)
        k = int(g["ks"][2]) if len(g["ks"]) >= 3 else int(g["ks"][-1])
        est = sx.estimate_walk_length(idx, model, 0.05, k, seed=int(c))
        np.testing.assert_array_equal(sorted(est.sampled), g[f"km{c}_est_ids"])
        if name == "intties":
            continue  # see test_walks_match_reference
        np.testing.assert_allclose([est.mean_visited, est.ci_low, est.ci_high, est.sample_size],
                                   g[f"km{c}_est"], rtol=1e-12)


def test_known_answers(sx):
    # tie -> lower id (reference tests/test_brute.py:18-26)
    m = sx.ModelPair(sx.FactorMatrix(np.array([[1.0, 0.0]])),
                     sx.FactorMatrix(np.array([[0.0, 1.0], [1.0, 0.0], [1.0, 1.0]])))
    for fn in (sx.topk_naive, sx.topk_matmul):
        r = fn(m, 1)[0]
        assert r.item_ids.tolist() == [1] and r.scores[0] == 1.0
    # norm-ordered list (tests/test_index.py:67-77)
    d = np.array([1.0, 1.0]) / np.sqrt(2.0)
    m = sx.ModelPair(sx.FactorMatrix(np.array([[1.0, 0.0], [0.0, 1.0]])),
                     sx.FactorMatrix(np.vstack([3.0 * d, 1.0 * d, 2.0 * d])))
    idx = sx.build_index(m, sx.kmeans(m.users, 1, seed=0))
    assert idx.item_ids[0].tolist() == [0, 2, 1]
    np.testing.assert_allclose(idx.bounds[0], [3.0, 2.0, 1.0], rtol=1e-12)
    # theta_b goldens (tests/test_clustering.py:86-112)
    th = sx.compute_max_angles(np.array([[1.0, 0.0], [0.0, 1.0]]), np.array([[0.5, 0.5]]), np.array([0, 0]))
    assert th[0] == pytest.approx(np.pi / 4, abs=1e-12)
    th = sx.compute_max_angles(np.array([[0.0, 0.0], [1.0, 0.0]]), np.array([[1.0, 0.0]]), np.array([0, 0]))
    assert th[0] == pytest.approx(np.pi)
    th = sx.compute_max_angles(np.array([[1.0, 2.0], [3.0, -1.0]]), np.array([[1.0, 2.0], [3.0, -1.0]]),
                               np.array([0, 1]))
    np.testing.assert_allclose(th, [0.0, 0.0], atol=1e-9)
    # two-point fixed point (tests/test_clustering.py:41-46)
    pts = np.array([[1.0, 1.0]] * 6 + [[5.0, -3.0]] * 4)
    cl = sx.kmeans(sx.FactorMatrix(pts), 2, seed=3)
    assert {tuple(c) for c in cl.centroids.values} == {(1.0, 1.0), (5.0, -3.0)}
    # duplicates: no empty clusters (tests/test_clustering.py:76-79)
    cl = sx.kmeans(sx.FactorMatrix(np.tile([[2.0, 2.0]], (9, 1))), 3, seed=0)
    assert all(ms.size > 0 for ms in cl.members)


def test_zero_slack_visits_exactly_k(sx):
    model = sx.generate_synthetic(sx.SyntheticSpec(3, 400, 8, seed=10, archetype_count=3))
    cl = sx.kmeans(model.users, 3, seed=0)
    idx = sx.build_index(model, cl)
    for uid in range(3):
        for k in (1, 5, 20):
            assert sx.query_user(idx, model, uid, k).visited == k


def test_zero_norm_user_and_item(sx):
    users = sx.FactorMatrix(np.vstack([np.zeros(4), np.ones(4)]))
    items = sx.FactorMatrix(np.random.default_rng(0).normal(size=(30, 4)))
    model = sx.ModelPair(users, items)
    idx = sx.build_index(model, sx.kmeans(model.users, 2, seed=0))
    r = sx.query_user(idx, model, 0, 5)
    assert r.item_ids.tolist() == [0, 1, 2, 3, 4] and np.all(r.scores == 0.0)
    users = sx.FactorMatrix(np.array([[1.0, 0.0], [0.8, 0.3]]))
    items = sx.FactorMatrix(np.array([[2.0, 1.0], [0.0, 0.0], [-1.0, 0.5]]))
    model = sx.ModelPair(users, items)
    idx = sx.build_index(model, sx.kmeans(model.users, 1, seed=0))
    pos = int(np.flatnonzero(idx.item_ids[0] == 1)[0])
    assert idx.bounds[0][pos] == 0.0


def test_k_beyond_item_count(sx):
    g = load_golden("syn1")
    model = _model(sx, g)
    n = model.num_items
    for fn in (sx.topk_naive, sx.topk_matmul):
        res = fn(model, n + 50)
        assert res[3].item_ids.size == n
    idx = sx.build_index(model, _ref_clustering(sx, g, 4), 64)
    want_ids, want_sc = __import__("simdex_oracle").topk_naive(g["users"], g["items"], n)
    for uid in (0, 17, 101):
        r = sx.query_user(idx, model, uid, n)
        assert_same_topk(r.item_ids, r.scores, want_ids[uid], want_sc[uid])


def test_query_batch_contract(sx):
    g = load_golden("syn1")
    model = _model(sx, g)
    idx = sx.build_index(model, _ref_clustering(sx, g, 4), 64)
    res = sx.query_batch(idx, model, [40, 3, 199, 3], 4)
    assert [r.user_id for r in res] == [40, 3, 199, 3]
    cached = sx.query_user(idx, model, 5, 4)
    res = sx.query_batch(idx, model, [5, 6], 4, precomputed={5: cached})
    assert res[0] is cached
    # the optimizer's sample map: built lazily, every lookup the same object,
    # and a serve that reuses it returns those objects at the sampled users
    est = sx.estimate_walk_length(idx, model, 0.1, 4, seed=3)
    some = sorted(est.sampled)[:5]
    assert est.sampled[some[0]] is est.sampled[some[0]]
    assert some[1] in est.sampled and -1 not in est.sampled and len(est.sampled) == len(list(est.sampled))
    with pytest.raises(KeyError):
        est.sampled[model.num_users + 7]
    full = sx.query_batch(idx, model, None, 4, precomputed=est.sampled)
    for u in some:
        assert full[u] is est.sampled[u]
        np.testing.assert_array_equal(full[u].item_ids, full.item_ids[u])
    sub = sx.query_batch(idx, model, [some[2], 0, some[2]], 4, precomputed=est.sampled)
    assert sub[0] is est.sampled[some[2]] and sub[2] is sub[0]
    with pytest.raises(ValueError):
        sx.query_user(idx, model, 0, 0)
    with pytest.raises(ValueError):
        sx.query_user(idx, model, 10_000, 1)
    with pytest.raises(ValueError):
        sx.query_batch(idx, model, [10_000], 1)


def test_query_vector_scale_invariance_and_exactness(sx):
    g = load_golden("syn1")
    model = _model(sx, g)
    idx = sx.build_index(model, _ref_clustering(sx, g, 4), 64)
    rng = np.random.default_rng(31)
    for _ in range(20):
        uid = int(rng.integers(0, model.num_users))
        alpha = float(rng.uniform(1e-3, 10.0))
        base = sx.query_user(idx, model, uid, 10)
        scaled = sx.query_vector(idx, model, alpha * model.users.values[uid], 10)
        assert np.array_equal(base.item_ids, scaled.item_ids)
        np.testing.assert_allclose(scaled.scores, alpha * base.scores, rtol=1e-9, atol=1e-12)
    ids = np.arange(model.num_items)
    for _ in range(10):
        v = rng.normal(size=model.factors) * rng.uniform(0.1, 4.0)
        r = sx.query_vector(idx, model, v, 7)
        assert np.array_equal(r.item_ids, np.lexsort((ids, -(model.items.values @ v)))[:7])
    with pytest.raises(sx.DimensionMismatchError):
        sx.query_vector(idx, model, [1.0, 2.0], 3)


def test_mutations_stay_exact(sx):
    import simdex_oracle as oracle
    g = load_golden("syn1")
    model = _model(sx, g)
    idx = sx.build_index(model, _ref_clustering(sx, g, 4), 64)
    dup = model.items.values[33].copy()
    idx2, model2 = sx.insert_item(idx, model, dup)
    new_id = model.num_items
    for c in range(idx2.num_clusters):
        a = int(np.flatnonzero(idx2.item_ids[c] == 33)[0])
        b = int(np.flatnonzero(idx2.item_ids[c] == new_id)[0])
        assert b == a + 1
    idx3, model3 = sx.insert_item(idx2, model2, np.full(model.factors, 0.7))
    want, _ = oracle.topk_naive(model3.users.values, model3.items.values, 6)
    for ws in (True, False):
        got = _ids(sx.query_batch(idx3, model3, None, 6, work_sharing=ws))
        np.testing.assert_array_equal(canonical_ids(model3.items.values, got),
                                      canonical_ids(model3.items.values, want))
    idx4, model4, fits = sx.add_user(idx, model, model.users.values[0].copy())
    assert fits is True and np.array_equal(idx4.item_ids, idx.item_ids)
    out = np.full(model.factors, -3.0)
    idx5, model5, fits = sx.add_user(idx, model, out)
    c = int(idx5.clustering.assignment[-1])
    if not fits:
        assert idx5.clustering.max_angle[c] > idx.clustering.max_angle[c]
    want, _ = oracle.topk_naive(model5.users.values, model5.items.values, 5)
    r = sx.query_user(idx5, model5, model5.num_users - 1, 5)
    np.testing.assert_array_equal(r.item_ids, want[-1])


def test_add_user_after_cached_serve(sx):
    """a query_batch(None) before add_user must not leave a
    cached all-users grouping that hides the new user afterwards."""
    import simdex_oracle as oracle
    g = load_golden("syn1")
    model = _model(sx, g)
    idx = sx.build_index(model, _ref_clustering(sx, g, 4), 64)
    before = sx.query_batch(idx, model, None, 5)
    assert len(before) == model.num_users
    for vec in (model.users.values[3].copy(), np.full(model.factors, -3.0)):  # fits / drifts
        idx2, model2, _ = sx.add_user(idx, model, vec)
        after = sx.query_batch(idx2, model2, None, 5)
        assert len(after) == model2.num_users == model.num_users + 1
        want, _ = oracle.topk_naive(model2.users.values, model2.items.values, 5)
        np.testing.assert_array_equal(after[-1].item_ids, want[-1])
        np.testing.assert_array_equal(after.item_ids[:, :], want)
        again = sx.query_batch(idx, model, None, 5)  # the original index still serves its own users
        assert len(again) == model.num_users


def test_band_overflow_falls_back_exactly(sx):
    """Hundreds of exactly tied items overflow every row's candidate buffer:
    the device-counted exact fallback must produce the reference ordering
    (score desc, id asc) on both the brute-force and the work-sharing path."""
    import simdex_oracle as oracle
    rng = np.random.default_rng(5)
    f = 24
    items = rng.normal(size=(900, f))
    items[100:700] = items[50]  # 601 copies of one vector
    users = rng.normal(size=(300, f))
    users[:150] = items[50] * rng.uniform(0.5, 2.0, size=(150, 1))  # these users rank the copies first
    model = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
    want, want_sc = oracle.topk_naive(users, items, 20)
    res = sx.topk_matmul(model, 20)
    np.testing.assert_array_equal(res.item_ids, want)
    np.testing.assert_allclose(res.scores, want_sc, rtol=1e-9, atol=1e-9)
    cl = sx.kmeans(model.users, 3, max_iters=5, seed=2)
    idx = sx.build_index(model, cl, 256)
    for ws in (True, False):
        out = sx.query_batch(idx, model, None, 20, work_sharing=ws)
        np.testing.assert_array_equal(out.item_ids, want)
        walked = [sx.query_user(idx, model, u, 20).visited for u in (0, 1, 200, 299)]
        if not ws:
            assert [int(out.visited[u]) for u in (0, 1, 200, 299)] == walked


def test_sidecar_round_trip(sx, tmp_path):
    g = load_golden("syn1")
    model = _model(sx, g)
    idx = sx.build_index(model, _ref_clustering(sx, g, 4), 64)
    sx.save_index(idx, tmp_path / "m.idx")
    back = sx.load_index(tmp_path / "m.idx")
    assert np.array_equal(back.item_ids, idx.item_ids) and np.array_equal(back.bounds, idx.bounds)
    assert back.block_size == 64
    for uid in (0, 50, 150):
        a, b = sx.query_user(back, model, uid, 3), sx.query_user(idx, model, uid, 3)
        assert np.array_equal(a.item_ids, b.item_ids) and a.visited == b.visited


def test_pipeline_branches_agree(sx):
    import simdex_oracle as oracle
    model = sx.generate_synthetic(sx.SyntheticSpec(180, 420, 8, seed=6))
    want, _ = oracle.topk_naive(model.users.values, model.items.values, 7)
    res_i, rep_i = sx.run_pipeline(model, k=7, num_clusters=6, block_size=64, seed=2, force="index")
    res_m, rep_m = sx.run_pipeline(model, k=7, num_clusters=6, block_size=64, seed=2, force="matmul")
    assert rep_i.decision == sx.INDEX and rep_m.decision == sx.MATMUL
    np.testing.assert_array_equal(_ids(res_i), want)
    np.testing.assert_array_equal(_ids(res_m), want)
    stages = dict(rep_i.csv_rows())
    assert {"cluster", "build", "estimate", "serve", "total", "decision"} <= set(stages)
    _, rep = sx.run_pipeline(sx.generate_synthetic(sx.SyntheticSpec(5, 40, 4, seed=8, archetype_count=5)), k=2)
    assert rep.num_clusters == 5


def test_heap_ops_grow_with_k(sx):
    model = sx.generate_synthetic(sx.SyntheticSpec(60, 250, 6, seed=6))
    totals = []
    for k in (1, 5, 10, 50):
        cnt = {}
        sx.topk_matmul(model, k, counters=cnt)
        totals.append(int(cnt["heap_ops"].sum()))
    assert totals == sorted(totals) and totals[0] < totals[-1]


def test_cfg1_full_size(sx):
    """BASELINE cfg1 (8192 x 2048, f=32, K=10): all users vs the reference's topk_naive."""
    from paper_1706_01449_b200 import workloads as W
    w = W.cfg1()
    g = load_golden("cfg1_k10")
    model = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    for fn in (sx.topk_matmul, sx.topk_naive):
        res = fn(model, 10)
        assert_same_topk(_ids(res), _scores(res), g["ids"].astype(np.int64), g["scores"], ctx=fn.__name__)


def test_query_set_setup_reuse(sx):
    """Query sets served repeatedly on their own contexts skip the
    per-query-set setup (simdex_ctx_set_query_token): alternating two sets,
    two depths, the all-users serve and a caller context reused across sets
    all give exactly the answers of a serve that rebuilds the setup."""
    import os
    from paper_1706_01449_b200 import _lib
    from paper_1706_01449_b200 import index as I
    rng = np.random.default_rng(5)
    users = rng.normal(size=(3000, 24)) * rng.lognormal(0, 0.5, size=(3000, 1))
    items = rng.normal(size=(5000, 24)) * rng.lognormal(0, 0.5, size=(5000, 1))
    m = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
    idx = sx.build_index(m, sx.kmeans(m.users, 12, max_iters=4, seed=1), 512)
    a = I.QuerySet(idx, rng.choice(3000, 700, replace=False))
    b = I.QuerySet(idx, np.arange(0, 3000, 3))
    shared = _lib.Context()

    def serve(q, k, ctx=None):
        return [t.cpu().numpy() for t in I.query_batch_tensors(idx, m, q, k, ctx=ctx)]

    os.environ["SIMDEX_NO_SETUP_REUSE"] = "1"
    try:
        want = {(n, k): serve(q, k) for n, q in (("a", a), ("b", b), ("all", None)) for k in (10, 5)}
    finally:
        del os.environ["SIMDEX_NO_SETUP_REUSE"]
    for _ in range(2):
        for n, q in (("a", a), ("b", b), ("all", None)):
            for k in (10, 5, 10):
                for got, exp in zip(serve(q, k), want[(n, k)]):
                    np.testing.assert_array_equal(got, exp)
                if q is not None:
                    for got, exp in zip(serve(q, k, ctx=shared.handle), want[(n, k)]):
                        np.testing.assert_array_equal(got, exp)
