"""World-size-2 tests of the multi-GPU plumbing on CPU (gloo): shard ranges,
global id offsets, the all-gather exchange of partial top-K lists and their
merge (the device merge kernel is replaced by the oracle's merge here; the
GPU test below runs the real kernel)."""

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
