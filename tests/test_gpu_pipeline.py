"""Full-size Algorithm 2 on the GPU: the decisions BASELINE.json requires,
the cfg4 answers pinned to the reference's (tests/golden/cfg4_sample.npz,
written by oracle/make_golden.py --cfg4 from the reference package run on
the GPU clustering), and the h0 calibration entry points
(optimizer.py:69-102, brute.py:116-150) on the device."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, assert_same_topk, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_01449_b200 as pkg
    return pkg


def _subsample_exact(users, items, k, sample):
    s = users[sample] @ items.T
    ids = np.stack([np.lexsort((np.arange(items.shape[0]), -row))[:k] for row in s])
    return ids, np.take_along_axis(s, ids, axis=1)


def test_cfg3_pipeline_picks_blocked_product(sx):
    """BASELINE configs[2]: "The cost optimizer must select blocked MM" --
    run_pipeline clusters (C=8, the default), estimates and decides matmul,
    and serves exact results."""
    from paper_1706_01449_b200 import workloads as W
    w = W.cfg3()
    m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    res, rep = sx.run_pipeline(m, k=10, num_clusters=8, max_iters=100, seed=w.seed)
    assert rep.decision == "matmul" and not rep.forced
    assert rep.estimate.pruning_fraction > rep.estimate.hw_factor
    sample = np.sort(np.random.default_rng(3).choice(m.num_users, 300, replace=False))
    want_ids, want_sc = _subsample_exact(m.users.values, m.items.values, 10, sample)
    np.testing.assert_allclose(res.scores[sample], want_sc, rtol=1e-9, atol=1e-9)
    same = (res.item_ids[sample] == want_ids).all(axis=1)
    assert same.mean() > 0.99  # rows that differ are exact near-ties (checked in test_gpu_large)


def test_cfg4_pipeline_picks_index(sx):
    """BASELINE configs[3] (index path): run_pipeline at the R2 shape with
    C=1024 decides the index and serves exact results."""
    from paper_1706_01449_b200 import workloads as W
    w = W.cfg4()
    m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    res, rep = sx.run_pipeline(m, k=10, num_clusters=1024, max_iters=3, seed=w.seed)
    assert rep.decision == "index" and not rep.forced
    assert len(res) == m.num_users
    sample = np.sort(np.random.default_rng(4).choice(m.num_users, 200, replace=False))
    want_ids, want_sc = _subsample_exact(m.users.values, m.items.values, 10, sample)
    np.testing.assert_allclose(res.scores[sample], want_sc, rtol=1e-9, atol=1e-9)
    assert (res.item_ids[sample] == want_ids).all(axis=1).mean() > 0.99


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "cfg4_sample.npz")), reason="no cfg4 fixture")
def test_cfg4_against_reference_on_gpu_clustering(sx):
    """cfg4 at full size: the GPU k-means reproduces the clustering the
    fixture was made from (bitwise), and on it the reference's own
    build_index / query_batch / query_user answers (ids, scores, visited,
    with and without work sharing, K = 1 and 10) for a 500-user sample."""
    import hashlib
    from paper_1706_01449_b200 import workloads as W
    g = load_golden("cfg4_sample")
    w = W.cfg4()
    m = sx.ModelPair(sx.FactorMatrix(w.users), sx.FactorMatrix(w.items))
    cl = sx.kmeans(m.users, 1024, max_iters=3, seed=w.seed)
    np.testing.assert_array_equal(cl.centroids.values, g["centroids"])
    sha = hashlib.sha256(np.asarray(cl.assignment).astype("<i8").tobytes()).digest()
    assert sha == g["assignment_sha"].tobytes()
    np.testing.assert_allclose(cl.max_angle, g["theta"], rtol=1e-12, atol=1e-15)
    idx = sx.build_index(m, cl, 4096)
    sample = g["sample"]
    for k in (1, 10):
        res = sx.query_batch(idx, m, sample, k, work_sharing=True)
        assert_same_topk(res.item_ids, res.scores, g[f"ws_k{k}_ids"].astype(np.int64), g[f"ws_k{k}_scores"],
                         ctx=f"cfg4 ws k={k}")
        np.testing.assert_array_equal(res.visited, g[f"ws_k{k}_visited"])
        nows = sx.query_batch(idx, m, sample, k, work_sharing=False)
        np.testing.assert_array_equal(nows.item_ids, g[f"nows_k{k}_ids"])
        np.testing.assert_array_equal(nows.visited, g[f"nows_k{k}_visited"])
        # the serving pass's ceiling exit (on for short walks) gives the same answers
        from paper_1706_01449_b200 import index as I
        I.note_walk_estimate(idx, k, 0.0)
        res2 = sx.query_batch(idx, m, sample, k, work_sharing=True)
        np.testing.assert_array_equal(res2.item_ids, res.item_ids)
        np.testing.assert_array_equal(res2.visited, res.visited)
        idx._dev.pop(("walk_estimate", k))


def test_calibration_entry_points(sx, tmp_path):
    """measure_throughput / _perpair_scan / calibrate_h0 on the device: both
    rates positive, the per-pair scan returns the exact answer it scores,
    h0 is the median rate ratio and persists as h0= in the config file."""
    import torch
    from paper_1706_01449_b200 import brute, optimizer
    spec = sx.SyntheticSpec(4000, 3000, 32, archetype_count=8, angular_spread=0.3, seed=5)
    m = sx.generate_synthetic(spec)
    s = sx.measure_throughput(m, k=10)
    assert s.blocked_rate > 0 and s.unblocked_rate > 0
    assert s.blocked_rate > s.unblocked_rate  # the tensor-core product beats the per-pair loop
    # _perpair_scan: the unpruned list walk visits every item and finds the exact top-K
    ids, bounds = brute._scan_list(m)
    from paper_1706_01449_b200 import _device, _ops
    q = torch.arange(m.num_users, dtype=torch.int64, device=ids.device)
    qc = torch.zeros(m.num_users, dtype=torch.int32, device=ids.device)
    oi, os_, ov = _ops.walk(_device.f64(m.users), _device.norms(m.users), _device.f64(m.items), ids, bounds, q, qc, 10,
                            no_prune=True)
    assert int(ov.min()) == int(ov.max()) == m.num_items
    want = sx.topk_naive(m, 10)
    np.testing.assert_array_equal(oi.cpu().numpy(), want.item_ids)
    path = tmp_path / "calib.conf"
    h0 = optimizer.calibrate_h0(m, k=10, repeats=3, config_path=path)
    assert 0.0 < h0 < 1.0
    assert optimizer.load_config(path)["h0"] == pytest.approx(h0)
    os.environ[optimizer.CONFIG_ENV] = str(path)
    try:
        assert optimizer.resolve_h0() == pytest.approx(h0)
    finally:
        del os.environ[optimizer.CONFIG_ENV]


def test_graph_replay_equals_eager(sx):
    """graphs.GraphedCall: the captured serving call (work-sharing query of a
    fixed query set; blocked product) replays to the eager answer."""
    import torch
    from paper_1706_01449_b200 import graphs, index as I, sharding
    spec = sx.SyntheticSpec(6000, 3000, 24, archetype_count=12, angular_spread=0.3, seed=9)
    m = sx.generate_synthetic(spec)
    cl = sx.kmeans(m.users, 10, max_iters=5, seed=1)
    idx = sx.build_index(m, cl, 512)
    shard = sharding.IndexShard(idx, m, 1, 3)
    for fn in (lambda: I.query_batch_tensors(idx, m, None, 10), lambda: shard.topk_tensors(7),
               lambda: sx.brute.topk_matmul_tensors(m, 5)[:2]):
        eager = [t.clone() for t in fn()]
        g = graphs.GraphedCall(fn)
        for _ in range(2):
            out = g()
            torch.cuda.synchronize()
            for a, b in zip(eager, out):
                assert torch.equal(a, b)


def test_graph_replay_survives_other_calls_and_arena_growth(sx):
    """Replays stay correct when other library calls run in between: the
    all-users query set serves on its own context (its captured setup is not
    disturbed by calls on the default context), and an arena a graph was
    captured over is retired, not freed, when a larger call outgrows it."""
    import torch
    from paper_1706_01449_b200 import graphs, index as I
    small = sx.generate_synthetic(sx.SyntheticSpec(3000, 1500, 16, archetype_count=8, angular_spread=0.3, seed=4))
    idx = sx.build_index(small, sx.kmeans(small.users, 6, max_iters=3, seed=1), 256)
    calls = [lambda: I.query_batch_tensors(idx, small, None, 10),        # own context from its second serve
             lambda: sx.brute.topk_matmul_tensors(small, 5)[:2]]         # the thread's default context
    eager = [[t.clone() for t in fn()] for fn in calls]
    graphed = [graphs.GraphedCall(fn) for fn in calls]
    # far larger calls on the default context: its arena is outgrown (or, if an
    # earlier test grew it, overwritten)
    big = sx.generate_synthetic(sx.SyntheticSpec(150000, 4000, 32, archetype_count=16, angular_spread=0.3, seed=5))
    sx.brute.topk_matmul_tensors(big, 20)
    idx_big = sx.build_index(big, sx.kmeans(big.users, 16, max_iters=2, seed=2), 1024)
    I.query_batch_tensors(idx_big, big, None, 20)
    scratch = torch.full((64 << 20,), 7, dtype=torch.int32, device="cuda")  # reuse any freed device memory
    torch.cuda.synchronize()
    for _ in range(2):
        for g, want in zip(graphed, eager):
            out = g()
            torch.cuda.synchronize()
            for a, b in zip(want, out):
                assert torch.equal(a, b)
    del scratch
