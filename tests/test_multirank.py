"""World-size-2 tests of the multi-GPU paths (sharding.py).

CPU (gloo, two processes): shard ranges, the cluster-routed user partition,
global id offsets, both exchanges of partial top-K lists (all-gather and the
per-user-slice all-to-all) with the oracle standing in for the device
compute.  GPU (marked): the same two-rank runs with the real CUDA partial
top-K, the device merge kernel and the index serve -- two processes on one
GPU whose exchange goes through gloo on host copies (their kernels never
wait on each other)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1706_01449_b200 import sharding


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def oracle_merge(gi, gs, k):
    """(score desc, id asc) merge of [world, U, kk] partial lists (CPU)."""
    w, u, kk = gi.shape
    ids = gi.permute(1, 0, 2).reshape(u, w * kk).numpy()
    sc = gs.permute(1, 0, 2).reshape(u, w * kk).numpy()
    out_i = np.empty((u, k), dtype=np.int32)
    out_s = np.empty((u, k))
    for r in range(u):
        order = np.lexsort((np.where(ids[r] < 0, np.iinfo(np.int32).max, ids[r]), -sc[r]))[:k]
        out_i[r], out_s[r] = ids[r][order], sc[r][order]
    return torch.from_numpy(out_i), torch.from_numpy(out_s)


def _worker(rank, world, port, users, items, k, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import simdex_oracle as O
        lo, hi = sharding.shard_range(items.shape[0], rank, world)
        pid, psc = O.topk_naive(users, items[lo:hi], k)         # this rank's shard, local ids
        gi, gs = sharding.exchange_partials(torch.from_numpy(pid.astype(np.int32)), torch.from_numpy(psc), lo, k)
        ids, sc = oracle_merge(gi, gs, k)
        out.put((rank, ids.numpy(), sc.numpy(), (lo, hi)))
    finally:
        dist.destroy_process_group()


def _guarded(target, rank, world, port, q, *args):
    """Run a rank body; report an exception through the queue instead of
    leaving the parent waiting."""
    import traceback
    try:
        target(rank, world, port, q, *args)
    except BaseException:  # noqa: BLE001
        q.put((rank, "error", traceback.format_exc()))
        raise


def _run_world(target, args, world=2, timeout=300):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_guarded, args=(target, r, world, port, q) + tuple(args)) for r in range(world)]
    for p in procs:
        p.start()
    got = []
    for _ in range(world):
        item = q.get(timeout=timeout)
        if len(item) == 3 and isinstance(item[1], str) and item[1] == "error":
            for p in procs:
                p.kill()
            raise AssertionError(f"rank {item[0]} failed:\n{item[2]}")
        got.append(item)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(got, key=lambda x: x[0])


def _a2a_worker(rank, world, port, out, users, items, k):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import simdex_oracle as O
        lo, hi = sharding.shard_range(items.shape[0], rank, world)
        if hi > lo:
            pid, psc = O.topk_naive(users, items[lo:hi], k)
        else:  # empty item shard: padded partial
            pid, psc = np.full((users.shape[0], 0), -1), np.zeros((users.shape[0], 0))
        k_eff = min(k, items.shape[0])
        gi, gs = sharding.exchange_user_slices(torch.from_numpy(pid.astype(np.int32)), torch.from_numpy(psc), lo,
                                               k_eff)
        ids, sc = oracle_merge(gi, gs, k_eff)
        out.put((rank, ids.numpy(), sc.numpy(), sharding.shard_range(users.shape[0], rank, world)))
    finally:
        dist.destroy_process_group()


def test_catalog_sharded_all_to_all_world2():
    """Each rank receives only its user slice's partial lists; the merged
    slices equal the single-process exact top-K (cross-shard tie included),
    also when one item shard is empty."""
    import simdex_oracle as O
    rng = np.random.default_rng(4)
    users = rng.normal(size=(41, 5))
    items = rng.normal(size=(90, 5)) * rng.lognormal(0, 0.7, (90, 1))
    items[70] = items[2]
    for it, k in ((items, 6), (items[:1], 3)):
        want_ids, want_sc = O.topk_naive(users, it, k)
        for rank, ids, sc, (lo, hi) in _run_world(_a2a_worker, (users, it, k)):
            np.testing.assert_array_equal(ids, want_ids[lo:hi])
            np.testing.assert_allclose(sc, want_sc[lo:hi], rtol=1e-12)


def _index_worker(rank, world, port, out, users, items, k, c, block):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import simdex_oracle as O
        cl = O.kmeans(users, c, 10, 1)
        ids, bounds, _ = O.build_index(items, cl["centroids"], cl["max_angle"])
        order, cuts = sharding.partition_users_by_cluster(cl["assignment"], c, world)
        mine = order[cuts[rank]:cuts[rank + 1]]
        got = O.query_batch((ids, bounds, cl["assignment"]), items, users, list(mine), k, block)
        # gather every rank's (user ids, top-K ids) on every rank over gloo
        n = torch.tensor([mine.size])
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, n)
        mx = int(max(x.item() for x in sizes))
        pad_u = torch.full((mx,), -1, dtype=torch.int64)
        pad_u[:mine.size] = torch.from_numpy(mine)
        pad_i = torch.full((mx, k), -1, dtype=torch.int64)
        pad_i[:mine.size] = torch.from_numpy(np.stack([np.asarray(g[0], dtype=np.int64) for g in got]))
        gu = [torch.empty_like(pad_u) for _ in range(world)]
        gi = [torch.empty_like(pad_i) for _ in range(world)]
        dist.all_gather(gu, pad_u)
        dist.all_gather(gi, pad_i)
        out.put((rank, torch.cat(gu).numpy(), torch.cat(gi).numpy(), cl["assignment"]))
    finally:
        dist.destroy_process_group()


def test_index_path_routed_by_cluster_world2():
    """Users sorted by cluster and cut in two: each rank serves its users on
    the (replicated) index; the union covers every user once and equals the
    single-process answer."""
    import simdex_oracle as O
    rng = np.random.default_rng(8)
    centers = rng.normal(size=(5, 6))
    users = centers[rng.integers(0, 5, 160)] + 0.2 * rng.normal(size=(160, 6))
    items = rng.normal(size=(120, 6))
    k = 4
    want, _ = O.topk_naive(users, items, k)
    for rank, gu, gi, assign in _run_world(_index_worker, (users, items, k, 5, 32)):
        live = gu >= 0
        assert np.array_equal(np.sort(gu[live]), np.arange(users.shape[0]))
        np.testing.assert_array_equal(gi[live], want[gu[live]])
        # contiguous in (cluster, id) order
        lab = assign[gu[live]]
        assert np.all(np.diff(lab) >= 0)


def test_partition_balances_estimated_work():
    from types import SimpleNamespace
    rng = np.random.default_rng(2)
    assign = rng.integers(0, 16, 10_000)
    costs = rng.uniform(1.0, 50.0, 16)
    for world in (1, 2, 3, 8):
        order, cuts = sharding.partition_users_by_cluster(assign, 16, world, costs)
        assert cuts[0] == 0 and cuts[-1] == assign.size and np.all(np.diff(cuts) >= 0)
        assert np.array_equal(np.sort(order), np.arange(assign.size))
        lab = assign[order]
        assert np.all(np.diff(lab) >= 0)
        shares = [costs[lab[cuts[r]:cuts[r + 1]]].sum() for r in range(world)]
        assert max(shares) - min(shares) <= 2 * costs.max() + 1e-9  # each cut is off by < one user
    # cluster_costs: continuation rates from the walk sample, shrunk to the global rate
    idx = SimpleNamespace(num_clusters=3, block_size=10, clustering=SimpleNamespace(assignment=np.array([0, 0, 1, 2])))
    res = SimpleNamespace(visited=np.array([10, 40, 10, 10]))
    est = SimpleNamespace(sampled=SimpleNamespace(user_ids=np.array([0, 1, 2, 3]), _res=res))
    cst = sharding.cluster_costs(idx, 100, est, shrink=0.0)
    np.testing.assert_allclose(cst, [10 + 50.0, 10.0, 10.0])
    assert np.all(sharding.cluster_costs(idx, 100, None) == 10)


def test_shard_ranges_cover_exactly():
    for n in (1, 7, 100, 1_000_003):
        for world in (1, 2, 3, 8):
            spans = [sharding.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1


def test_catalog_sharded_exchange_world2():
    """Two gloo ranks, each with half of the catalogue: the all-gathered,
    merged partial lists equal the single-process exact top-K."""
    import simdex_oracle as O
    rng = np.random.default_rng(3)
    users = rng.normal(size=(40, 6))
    items = rng.normal(size=(101, 6)) * rng.lognormal(0, 0.7, (101, 1))
    items[77] = items[3]  # an exact tie across the two shards
    k = 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, users, items, k, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want_ids, want_sc = O.topk_naive(users, items, k)
    for rank, ids, sc, span in got:
        np.testing.assert_array_equal(ids, want_ids)
        np.testing.assert_allclose(sc, want_sc, rtol=1e-12)


@pytest.mark.gpu
def test_merge_kernel_matches_oracle_merge():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1706_01449_b200 import _ops
    rng = np.random.default_rng(5)
    w, u, kk = 4, 300, 16
    sc = np.sort(rng.normal(size=(w, u, kk)), axis=2)[:, :, ::-1].copy()
    sc[1, :, 3] = sc[0, :, 3]  # cross-shard score ties -> id order decides
    ids = np.stack([rng.permutation(10_000)[: u * kk].reshape(u, kk) + 10_000 * r for r in range(w)]).astype(np.int32)
    for r in range(w):  # order each partial list by (score desc, id asc) like the kernel's inputs
        for row in range(u):
            o = np.lexsort((ids[r, row], -sc[r, row]))
            ids[r, row], sc[r, row] = ids[r, row][o], sc[r, row][o]
    gi, gs = torch.from_numpy(ids), torch.from_numpy(sc)
    want_i, want_s = oracle_merge(gi, gs, 10)
    got_i, got_s = _ops.merge_topk(gi.cuda().contiguous(), gs.cuda().contiguous(), 10)
    np.testing.assert_array_equal(got_i.cpu().numpy(), want_i.numpy())
    np.testing.assert_array_equal(got_s.cpu().numpy(), want_s.numpy())


def _gpu_worker(rank, world, port, out, users, items, k, mode):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1706_01449_b200 as sx
        model = sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))
        if mode in ("all_to_all", "all_gather"):
            ids, sc, lo = sharding.catalog_sharded_topk(model, k, exchange=mode)
            out.put((rank, ids.cpu().numpy(), sc.cpu().numpy(), lo, None))
        elif mode == "users":
            shard = sharding.UserShard(model, rank, world)
            ids, sc = shard.topk_tensors(k)
            out.put((rank, ids.cpu().numpy(), sc.cpu().numpy(), shard.lo, None))
        else:  # index path, users routed by cluster
            cl = sx.kmeans(model.users, 12, max_iters=5, seed=1)
            idx = sx.build_index(model, cl, 256)
            est = sx.estimate_walk_length(idx, model, 0.05, k, seed=1)
            shard = sharding.IndexShard(idx, model, rank, world, est)
            ids, sc, vis = shard.topk_tensors(k)
            full = sx.query_batch(idx, model, None, k)
            out.put((rank, ids.cpu().numpy(), sc.cpu().numpy(), shard.user_ids,
                     (full.item_ids[shard.user_ids], full.visited[shard.user_ids], vis.cpu().numpy())))
    finally:
        dist.destroy_process_group()


def _gpu_model(seed=11, nu=3000, ni=2000, f=32):
    rng = np.random.default_rng(seed)
    centers = rng.normal(size=(12, f))
    users = (centers[rng.integers(0, 12, nu)] + 0.3 * rng.normal(size=(nu, f))).astype(np.float32).astype(np.float64)
    items = (rng.normal(size=(ni, f)) * rng.lognormal(0, 0.7, (ni, 1))).astype(np.float32).astype(np.float64)
    items[1500] = items[7]  # exact tie across the two item shards
    return users, items


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["all_to_all", "all_gather", "users"])
def test_sharded_blocked_product_real_kernels_world2(mode):
    """Two ranks (processes on one GPU, gloo exchange of host copies) with the
    real tensor-core partial top-K and device merge: catalogue sharding with
    either exchange, and contiguous user blocks; equal to the exact top-K."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import simdex_oracle as O
    users, items = _gpu_model()
    k = 10
    want_ids, want_sc = O.topk_naive(users, items, k)
    got = _run_world(_gpu_worker, (users, items, k, mode))
    for rank, ids, sc, lo, _ in got:
        n = ids.shape[0]
        if mode == "all_gather":
            assert lo == 0 and n == users.shape[0]
        np.testing.assert_array_equal(ids, want_ids[lo:lo + n])
        np.testing.assert_allclose(sc, want_sc[lo:lo + n], rtol=1e-9, atol=1e-9)
    if mode != "all_gather":
        assert sum(g[1].shape[0] for g in got) == users.shape[0]


@pytest.mark.gpu
def test_index_path_routed_by_cluster_real_kernels_world2():
    """Index path sharded by cluster over two ranks: every user served once,
    ids/scores exact, visited equal to the unsharded query_batch."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import simdex_oracle as O
    users, items = _gpu_model(seed=12)
    k = 10
    want_ids, want_sc = O.topk_naive(users, items, k)
    got = _run_world(_gpu_worker, (users, items, k, "index"))
    seen = np.concatenate([g[3] for g in got])
    assert np.array_equal(np.sort(seen), np.arange(users.shape[0]))
    for rank, ids, sc, uids, (full_ids, full_vis, vis) in got:
        np.testing.assert_array_equal(ids, want_ids[uids])
        np.testing.assert_allclose(sc, want_sc[uids], rtol=1e-9, atol=1e-9)
        np.testing.assert_array_equal(ids, full_ids)
        np.testing.assert_array_equal(vis, full_vis)
