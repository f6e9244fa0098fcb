"""BASELINE configurations at full size on the GPU, checked against an exact
float64 top-K of a uniform user subsample (the reference's own
_subsample_oracle_matches pattern, tests/test_acceptance.py:258-264): cfg3
(brute force, the optimizer's low-similarity case), cfg4 (index + work
sharing at the R2 shape, C=1024) and cfg5 (1M x 1M, f=128, K=100)."""

import numpy as np
import pytest

from conftest import near_tie_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_01449_b200 as pkg
    return pkg


def _exact_topk(users, items, k, extra=1):
    """Exact top-(k+extra) under (score desc, id asc), float64 GEMM in chunks;
    the extra column exposes near ties at the k-th position."""
    kk = min(k + extra, items.shape[0])
    ids = np.empty((users.shape[0], kk), dtype=np.int64)
    sc = np.empty((users.shape[0], kk))
    for a in range(0, users.shape[0], 64):
        s = users[a:a + 64] @ items.T
        part = np.argpartition(-s, kk - 1, axis=1)[:, :kk]
        kth = np.take_along_axis(s, part, axis=1).min(axis=1)
        for r in range(s.shape[0]):
            cand = np.flatnonzero(s[r] >= kth[r])          # everything tied with the k-th too
            order = np.lexsort((cand, -s[r, cand]))[:kk]   # score desc, id asc
            ids[a + r] = cand[order]
            sc[a + r] = s[r, cand[order]]
    return ids, sc


def _check(res_ids, res_scores, users, items, k, sample, ctx):
    want_ids, want_sc = _exact_topk(users[sample], items, k)
    got_ids = np.asarray(res_ids)[sample]
    got_sc = np.asarray(res_scores)[sample]
    k_eff = got_ids.shape[1]
    np.testing.assert_allclose(got_sc, want_sc[:, :k_eff], rtol=1e-9, atol=1e-9, err_msg=ctx)
    ties = near_tie_rows(want_sc, k_eff)
    bad = np.flatnonzero((got_ids != want_ids[:, :k_eff]).any(axis=1) & ~ties)
    assert bad.size == 0, f"{ctx}: {bad.size} rows differ, first {sample[bad[0]]}"


def test_cfg3_brute_force_full_size(sx):
    from paper_1706_01449_b200 import workloads as W
    w = W.cfg3()
    m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    res = sx.topk_matmul(m, 10)
    sample = np.sort(np.random.default_rng(0).choice(m.num_users, 2000, replace=False))
    _check(res.item_ids, res.scores, m.users.values, m.items.values, 10, sample, "cfg3 K=10")


@pytest.mark.parametrize("k", [1, 10])
def test_cfg4_index_work_sharing_full_size(sx, k):
    from paper_1706_01449_b200 import workloads as W
    w = W.cfg4()
    m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    cl = sx.kmeans(m.users, 1024, max_iters=3, seed=3)
    idx = sx.build_index(m, cl, 4096)
    res = sx.query_batch(idx, m, None, k, work_sharing=True)
    sample = np.sort(np.random.default_rng(1).choice(m.num_users, 2000, replace=False))
    _check(res.item_ids, res.scores, m.users.values, m.items.values, k, sample, f"cfg4 K={k}")
    vis = np.asarray(res.visited)
    assert (vis >= 4096).all() and (vis <= m.num_items).all()
    # with the walk estimate in place (short walks) the prefix pass exits on
    # the list ceilings: identical ids, scores and visited for every user
    est = sx.estimate_walk_length(idx, m, 0.001, k, seed=3)
    assert est.mean_visited < 0.3 * 4096
    res2 = sx.query_batch(idx, m, None, k, work_sharing=True)
    np.testing.assert_array_equal(np.asarray(res2.item_ids), np.asarray(res.item_ids))
    np.testing.assert_array_equal(np.asarray(res2.scores), np.asarray(res.scores))
    np.testing.assert_array_equal(np.asarray(res2.visited), vis)


def test_cfg5_catalogue_scale_full_size(sx):
    from paper_1706_01449_b200 import workloads as W
    w = W.cfg5()
    m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    res = sx.topk_matmul(m, 100)
    sample = np.sort(np.random.default_rng(2).choice(m.num_users, 256, replace=False))
    _check(res.item_ids, res.scores, m.users.values, m.items.values, 100, sample, "cfg5 K=100")


@pytest.mark.parametrize("k,ln_sigma", [(1, 1.0), (10, 1.0), (50, 0.7), (100, 1.5)])
def test_brute_force_early_exit_skewed_norms(sx, k, ln_sigma):
    """Log-normal item norms: the norm-sorted brute-force pass ends units early
    (every row's threshold above ||u|| times the remaining norms); results must
    equal the exact top-K for every user (60k users = 235 units over 148 SMs,
    so CTAs run several units and the end-of-unit handshake is exercised)."""
    rng = np.random.default_rng(k)
    users = rng.normal(0.0, 1.0, (60_000, 48)).astype(np.float32)
    items = rng.normal(0.0, 1.0, (40_000, 48))
    items = (items * rng.lognormal(0.0, ln_sigma, items.shape[0])[:, None]).astype(np.float32)
    m = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
    res = sx.topk_matmul(m, k)
    sample = np.sort(np.random.default_rng(1).choice(m.num_users, 1500, replace=False))
    _check(res.item_ids, res.scores, m.users.values, m.items.values, k, sample, f"skewed K={k}")


def test_catalog_sharded_shards_and_device_merge(sx):
    """cfg5's data path on one GPU: the catalogue split into 4 contiguous
    shards, each shard's exact top-100 by the tensor-core pass (early exit on
    its norm-sorted operand), global ids, padded, merged on the device
    (simdex_merge_topk) -- equal to the unsharded exact top-K."""
    import torch
    from paper_1706_01449_b200 import _ops, brute, sharding
    rng = np.random.default_rng(4)
    users = rng.normal(0.0, 1.0, (6_000, 128)).astype(np.float32)
    items = rng.normal(0.0, 1.0, (30_001, 128))
    items = (items * rng.lognormal(0.0, 0.7, items.shape[0])[:, None]).astype(np.float32)
    m = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
    k, world = 100, 4
    parts = []
    for r in range(world):
        part, off = sharding.item_shard(m, r, world)
        ids, sc, _ = brute.topk_matmul_tensors(part, k)
        parts.append(sharding.pad_partial(ids, sc, off, k))
    gi = torch.stack([p[0] for p in parts]).contiguous()
    gs = torch.stack([p[1] for p in parts]).contiguous()
    got_i, got_s = _ops.merge_topk(gi, gs, k)
    sample = np.sort(np.random.default_rng(0).choice(m.num_users, 400, replace=False))
    _check(got_i.cpu().numpy(), got_s.cpu().numpy(), m.users.values, m.items.values, k, sample, "sharded K=100")


def test_catalog_sharded_topk_nccl_single_rank(sx):
    """catalog_sharded_topk itself over a one-rank NCCL group (the all-to-all /
    all-gather and the merge run for real; two-rank runs: test_multirank.py)."""
    import os
    import torch
    import torch.distributed as dist
    from paper_1706_01449_b200 import sharding
    if dist.is_initialized():
        pytest.skip("a process group is already initialised")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29571")
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        rng = np.random.default_rng(6)
        users = rng.normal(0.0, 1.0, (3_000, 64)).astype(np.float32)
        items = rng.normal(0.0, 1.0, (9_000, 64)).astype(np.float32)
        m = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
        sample = np.sort(np.random.default_rng(1).choice(m.num_users, 300, replace=False))
        for exchange in ("all_to_all", "all_gather"):
            ids, sc, lo = sharding.catalog_sharded_topk(m, 20, exchange=exchange)
            assert lo == 0 and ids.shape[0] == m.num_users
            _check(ids.cpu().numpy(), sc.cpu().numpy(), m.users.values, m.items.values, 20, sample,
                   f"nccl world 1 {exchange}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("path", ["brute", "index"])
def test_heavy_tailed_user_norms_stay_exact(sx, path):
    """Users with log-normal(0, 3) norms span ~20 binades: with one matrix-wide
    fp16 scale the small rows would sink into subnormals, widen their band and
    overflow to the exact fallback.  The per-row scale keeps every row's band
    relative: results exact, and (almost) no row needs the fallback."""
    from paper_1706_01449_b200 import _lib
    rng = np.random.default_rng(17)
    nu, ni, f, k = 20_000, 6_000, 48, 10
    users = rng.normal(size=(nu, f)) * rng.lognormal(0.0, 3.0, (nu, 1))
    items = rng.normal(size=(ni, f)) * rng.lognormal(0.0, 0.5, (ni, 1))
    users = users.astype(np.float32).astype(np.float64)
    items = items.astype(np.float32).astype(np.float64)
    m = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
    if path == "brute":
        res = sx.topk_matmul(m, k)
    else:
        cl = sx.kmeans(m.users, 16, max_iters=5, seed=3)
        idx = sx.build_index(m, cl, 1024)
        res = sx.query_batch(idx, m, None, k)
    import torch
    torch.cuda.synchronize()
    fb = _lib.fallback_rows()
    print(f"{path}: fallback rows {fb} of {nu} ({fb / nu:.4%}), user norm range "
          f"{np.linalg.norm(users, axis=1).min():.2e} .. {np.linalg.norm(users, axis=1).max():.2e}")
    sample = np.sort(rng.choice(nu, 1500, replace=False))
    _check(res.item_ids, res.scores, users, items, k, sample, f"heavy-tailed norms {path}")
    assert fb <= nu // 1000


@pytest.mark.parametrize("k,mode", [(10, "hybrid"), (16, "hybrid"), (10, "list"), (12, "none"), (50, "hybrid")])
def test_work_sharing_prefix_layouts_and_list_catalogue_pass(sx, k, mode):
    """The prefix layouts of the work-sharing pass (centroid order without an
    exit, hybrid head + list order with the exit, list order with the exit)
    and the list-order catalogue pass (query sets of 50k+ users, K >= 8) give
    the exact top-K of every user, and visited = max(B', the walk's visited)
    (index.py:372-387) against the walk kernel without work sharing."""
    from paper_1706_01449_b200 import index as I
    rng = np.random.default_rng(7 + k)
    nu, ni, f, c = 64000, 6000, 32, 48
    centers = rng.normal(size=(c, f))
    users = centers[rng.integers(0, c, nu)] + rng.normal(0, 0.4, (nu, f))
    d = rng.normal(size=(ni, f))
    items = d / np.linalg.norm(d, axis=1, keepdims=True) * rng.lognormal(0, 0.5, (ni, 1))
    users, items = users.astype(np.float32).astype(np.float64), items.astype(np.float32).astype(np.float64)
    m = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
    block = 1024
    idx = sx.build_index(m, sx.kmeans(m.users, c, max_iters=3, seed=2), block)
    est = {"hybrid": 0.3, "list": 0.05, "none": 0.9}[mode] * block
    I.note_walk_estimate(idx, k, est)
    assert bool(I._ws_options(idx, k, ni, True)) == (mode != "none")
    if mode != "none":
        assert (I._prefix_head(idx, k, ni) > 0) == (mode == "hybrid")
    assert idx.device_full_lists(m) is not None  # (a serving index builds it after its first large batch)
    ids, sc, vis = (t.cpu().numpy() for t in I.query_batch_tensors(idx, m, None, k, work_sharing=True))
    sample = rng.choice(nu, 800, replace=False)
    _check(ids, sc, users, items, k, sample, f"{mode} K={k}")
    ids0, sc0, vis0 = (t.cpu().numpy() for t in I.query_batch_tensors(idx, m, None, k, work_sharing=False))
    np.testing.assert_array_equal(vis, np.maximum(min(block, ni), vis0))
    np.testing.assert_array_equal(ids, ids0)


def test_full_list_operand_is_built_after_the_first_large_batch(sx):
    """The list-order catalogue pass's operand is built once an index has
    served a large batch (index.FULL_LISTS_AFTER), not by build_index or a
    one-shot run_pipeline; the answers before and after are identical."""
    from paper_1706_01449_b200 import index as I
    rng = np.random.default_rng(3)
    nu, ni, f, c, k = 52000, 3000, 16, 24, 10
    centers = rng.normal(size=(c, f))
    users = (centers[rng.integers(0, c, nu)] + rng.normal(0, 0.5, (nu, f))).astype(np.float32).astype(np.float64)
    items = rng.normal(size=(ni, f)).astype(np.float32).astype(np.float64)
    m = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
    idx = sx.build_index(m, sx.kmeans(m.users, c, max_iters=2, seed=1), 512)
    assert "full_lists" not in idx._dev and "prefix" not in idx._dev
    first = [t.clone() for t in I.query_batch_tensors(idx, m, None, k)]
    assert "full_lists" not in idx._dev
    for _ in range(I.FULL_LISTS_AFTER):
        second = [t.clone() for t in I.query_batch_tensors(idx, m, None, k)]
    assert idx._dev.get("full_lists") is not None
    import torch
    for a, b in zip(first, second):
        assert torch.equal(a, b)


def test_all_user_serve_with_overlapped_copies_equals_one_batch(sx):
    """query_batch(None) serves large models in contiguous user ranges with
    the device->host copies overlapped; the results are those of one batch."""
    from paper_1706_01449_b200 import index as I
    rng = np.random.default_rng(11)
    nu, ni, f, c, k = 210000, 2500, 16, 16, 10
    centers = rng.normal(size=(c, f))
    users = (centers[rng.integers(0, c, nu)] + rng.normal(0, 0.5, (nu, f))).astype(np.float32).astype(np.float64)
    items = rng.normal(size=(ni, f)).astype(np.float32).astype(np.float64)
    m = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
    idx = sx.build_index(m, sx.kmeans(m.users, c, max_iters=2, seed=1), 512)
    assert I._d2h_parts(m, k) == 2
    for _ in range(3):  # (one batch first; then the ranges, whose second serve takes the list-order catalogue pass)
        res = sx.query_batch(idx, m, None, k)
    assert ("user_ranges", nu, 2) in idx._dev
    ids, sc, vis = (t.cpu().numpy() for t in I.query_batch_tensors(idx, m, None, k))
    np.testing.assert_array_equal(res.item_ids, ids)
    np.testing.assert_array_equal(res.scores, sc)
    np.testing.assert_array_equal(np.asarray(res.visited), vis)
    assert len(res) == nu and res[nu - 1].item_ids.tolist() == ids[-1].tolist()


@pytest.mark.parametrize("f", [34, 36, 38, 46, 48, 50, 62, 64, 66])
def test_cooperative_rescoring_factor_edges(sx, f):
    """finalize's cooperative rescoring (8 lanes share a candidate's item row,
    factor pairs 8 i + lane) at the edges of its range: f = 36..64 takes it,
    with the third and fourth pair of a lane present or not; 34 and 66 do not.
    Blocked product and work-sharing query against the exact float64 top-K,
    K = 1, 3, 10, 20; inside the range every (user, item) score has one
    arithmetic, so the two paths return bit-equal scores (outside it the
    summation order follows the row's survivor count: last-bit differences)."""
    from paper_1706_01449_b200 import index as I
    rng = np.random.default_rng(100 + f)
    nu, ni, c = 6000, 3000, 12
    centers = rng.normal(size=(c, f))
    users = (centers[rng.integers(0, c, nu)] + rng.normal(0, 0.5, (nu, f))).astype(np.float32).astype(np.float64)
    items = (rng.normal(size=(ni, f)) * rng.lognormal(0, 0.4, (ni, 1))).astype(np.float32).astype(np.float64)
    m = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
    idx = sx.build_index(m, sx.kmeans(m.users, c, max_iters=3, seed=2), 512)
    sample = np.arange(0, nu, 5)
    for k in (1, 3, 10, 20):
        b_ids, b_sc = (t.cpu().numpy() for t in sx.brute.topk_matmul_tensors(m, k)[:2])
        _check(b_ids, b_sc, users, items, k, sample, f"brute f={f} K={k}")
        ids, sc, _ = (t.cpu().numpy() for t in I.query_batch_tensors(idx, m, None, k))
        _check(ids, sc, users, items, k, sample, f"index f={f} K={k}")
        if 36 <= f <= 64:
            np.testing.assert_array_equal(sc, b_sc)
