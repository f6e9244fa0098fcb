"""Multi-GPU sharding of the serving path.

One process per GPU, ``torch.distributed`` for the plumbing.  Three layouts:

* **Blocked product, users sharded** (configs 1, 3; brute.py:59-113): rank r
  serves a contiguous block of users against the whole (replicated)
  catalogue.  Users are independent, so there is no data-path collective.
* **Index path, users routed by cluster** (configs 2, 4; PAPER.md:859-863
  "partition clusters across cores ... and route users based on their
  cluster assignments"): users are ordered by (cluster, id) -- the order of
  the clustering's member lists -- and cut into ``world`` contiguous ranges
  of equal estimated work.  A user's work is the prefix product (B' items)
  plus, when its walk runs past B', the catalogue pass; the per-cluster
  continuation rate comes from the optimizer's own walk sample
  (optimizer.py:117-145), shrunk toward the global rate for clusters with few
  samples.  Every rank holds the whole (read-only) index; no collective.
* **Catalogue sharded** (config 5): rank r scores ALL users against its
  contiguous item shard (certified tensor-core top-K), then one exchange:
  an all-to-all sends every rank the partial lists of ITS user slice only
  (each rank receives U/world x K x world entries instead of the all-gather's
  U x K x world), and a device merge by (score desc, global id asc)
  (simdex_merge_topk) gives the exact global top-K of that slice: every
  global top-K item is in its own shard's top-K.  Scores travel as float64
  (the reference's precision): a float32 exchange could merge two scores
  that differ below float32 resolution in the wrong order.

Collectives go through the group's backend: NCCL with device tensors, or
gloo with host copies (the CPU tests, and two processes sharing one GPU).
"""

from __future__ import annotations

import os

import numpy as np
import torch
import torch.distributed as dist

from . import _lib, _device, _ops, brute
from . import index as index_mod
from .model_io import FactorMatrix, ModelPair


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of ``n`` rows for ``rank``."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _rank_world(group=None, rank=None, world=None):
    if rank is None or world is None:
        return dist.get_rank(group), dist.get_world_size(group)
    return int(rank), int(world)


# ---------------------------------------------------------------------------
# blocked product: contiguous user blocks
# ---------------------------------------------------------------------------

def user_shard(model: ModelPair, rank: int, world: int) -> tuple[ModelPair, int]:
    """This rank's users (whole catalogue) and the global id of its first user."""
    lo, hi = shard_range(model.num_users, rank, world)
    return ModelPair(FactorMatrix(model.users.values[lo:hi]), model.items), lo


# concurrent serving calls per rank (IndexShard, UserShard), each on its own
# stream and context (SIMDEX_SHARD_PARTS overrides: A/B timing only)
_SHARD_PARTS = int(os.environ.get("SIMDEX_SHARD_PARTS", "2"))


class UserShard:
    """A rank's resident block of users for repeated blocked-product serving
    (the sub-model keeps its device copies between calls; when the parent
    model is already on the device, the block is a view of its rows).  At
    N > 1 the block is served as ``_SHARD_PARTS`` concurrent calls on their
    own streams and contexts (the last wave of units of one call leaves the
    GPU partly idle; see IndexShard)."""

    def __init__(self, model: ModelPair, rank: int, world: int, parts: int | None = None):
        self.model, self.lo = user_shard(model, rank, world)
        self.hi = self.lo + self.model.num_users
        _device.share_rows(model.users, self.model.users, self.lo, self.hi)
        n_parts = (_SHARD_PARTS if world > 1 else 1) if parts is None else parts
        nu = self.model.num_users
        self.parts, self.contexts, self.streams = [], [], []
        if n_parts > 1 and nu >= 1024 * n_parts:
            cuts = [nu * i // n_parts for i in range(n_parts + 1)]
            for a, b in zip(cuts[:-1], cuts[1:]):
                sub = ModelPair(FactorMatrix(self.model.users.values[a:b]), self.model.items)
                _device.share_rows(self.model.users, sub.users, a, b)
                self.parts.append(sub)
                self.contexts.append(_lib.Context())
                self.streams.append(torch.cuda.Stream())

    def topk_tensors(self, k: int):
        if not self.parts:
            ids, sc, _ = brute.topk_matmul_tensors(self.model, k)
            return ids, sc
        main = torch.cuda.current_stream()
        fork = torch.cuda.Event()
        fork.record(main)
        outs = []
        for sub, ctx, st in zip(self.parts, self.contexts, self.streams):
            st.wait_event(fork)
            with torch.cuda.stream(st):
                outs.append(brute.topk_matmul_tensors(sub, k, ctx=ctx.handle)[:2])
        for st in self.streams:
            join = torch.cuda.Event()
            join.record(st)
            main.wait_event(join)
        for o in outs:
            for t in o:
                t.record_stream(main)
        return tuple(torch.cat([o[i] for o in outs]) for i in range(2))

    def stats(self):
        """(users, 0, executed pairs, 0) summed over this rank's serving calls
        (after the stream synchronised)."""
        if not self.parts:
            return self.model.num_users, 0, _lib.executed_pairs()[0], 0
        return self.model.num_users, 0, sum(ctx.stats()[2] for ctx in self.contexts), 0


def user_sharded_topk(model: ModelPair, k: int, group=None, rank=None, world=None):
    """Exact top-K of this rank's contiguous user block (no collective).
    Returns (ids int32 [n_r, k_eff], scores float64, first user id)."""
    rank, world = _rank_world(group, rank, world)
    part, lo = user_shard(model, rank, world)
    ids, sc, _ = brute.topk_matmul_tensors(part, k)
    return ids, sc, lo


# ---------------------------------------------------------------------------
# index path: users routed by cluster
# ---------------------------------------------------------------------------

def cluster_costs(index, num_items: int, estimate=None, shrink: float = 2.0) -> np.ndarray:
    """Estimated work per user of each cluster, in scored items: B' for the
    prefix product plus |I| x the cluster's rate of walks running past B'.
    The rate is the walk sample's (``estimate.sampled``: visited per sampled
    user, optimizer.py:117-145), shrunk toward the global rate with weight
    ``shrink``; without an estimate every cluster costs the same."""
    c = index.num_clusters
    bp = min(index.block_size, num_items)
    if estimate is None or bp >= num_items:
        return np.full(c, float(bp))
    sampled = estimate.sampled
    uids = np.asarray(sampled.user_ids, dtype=np.int64)
    res = sampled._res if hasattr(sampled, "_res") else None
    vis = np.asarray(res.visited if res is not None else [sampled[int(u)].visited for u in uids], dtype=np.float64)
    cont = (vis > bp).astype(np.float64)
    lab = np.asarray(index.clustering.assignment)[uids]
    n_c = np.bincount(lab, minlength=c).astype(np.float64)
    k_c = np.bincount(lab, weights=cont, minlength=c)
    glob = float(cont.mean()) if cont.size else 0.0
    rate = (k_c + shrink * glob) / (n_c + shrink)
    return bp + rate * float(num_items)


def partition_users_by_cluster(assignment, num_clusters: int, world: int, costs=None):
    """Users in (cluster, id) order and ``world + 1`` cut points into that
    order, so that rank r's users ``order[cuts[r]:cuts[r+1]]`` carry an equal
    share of sum(costs[cluster(u)]) (cuts fall inside clusters when needed).
    Returns (order int64 [U], cuts int64 [world + 1])."""
    a = np.asarray(assignment, dtype=np.int64)
    order = np.argsort(a, kind="stable")
    w = np.ones(num_clusters) if costs is None else np.asarray(costs, dtype=np.float64)
    cum = np.cumsum(w[a[order]])
    total = float(cum[-1]) if cum.size else 0.0
    targets = total * np.arange(1, world) / world
    inner = np.searchsorted(cum, targets, side="left") + 1 if cum.size else np.zeros(world - 1, dtype=np.int64)
    cuts = np.concatenate([[0], np.minimum(inner, a.size), [a.size]]).astype(np.int64)
    return order, np.maximum.accumulate(cuts)


class IndexShard:
    """A rank's users for the index path: the cluster-routed range of the
    (cluster, id) order, prepared once (index.QuerySet) for repeated serving.

    At N > 1 a rank's share is small enough that one serving call leaves
    the GPU partly idle (the last wave of units, the catalogue pass of the
    few continuing users, the small setup kernels), so the share is cut into
    ``_SHARD_PARTS`` cost-balanced contiguous parts served concurrently, each
    on its own stream and execution context (fork / join by events, CUDA-graph
    capturable); their outputs concatenate to ``user_ids`` order."""

    def __init__(self, index, model: ModelPair, rank: int, world: int, estimate=None, parts: int | None = None):
        costs = cluster_costs(index, model.num_items, estimate)
        assign = np.asarray(index.clustering.assignment)
        order, cuts = partition_users_by_cluster(assign, index.num_clusters, world, costs)
        self.user_ids = order[cuts[rank]:cuts[rank + 1]]
        self.share = float(costs[assign[self.user_ids]].sum() / max(costs[assign].sum(), 1e-30))
        self.index, self.model = index, model
        n_parts = (_SHARD_PARTS if world > 1 else 1) if parts is None else parts
        if self.user_ids.size < 1024 * n_parts:
            n_parts = 1
        self.parts, self.contexts, self.streams = [], [], []
        self.queries = None
        if self.user_ids.size and n_parts == 1:
            self.queries = index_mod.QuerySet(index, self.user_ids)
        elif self.user_ids.size:
            cum = np.cumsum(costs[assign[self.user_ids]])
            inner = np.searchsorted(cum, cum[-1] * np.arange(1, n_parts) / n_parts, side="left") + 1
            pc = np.concatenate([[0], np.minimum(inner, self.user_ids.size), [self.user_ids.size]])
            pc = np.maximum.accumulate(pc)
            for a, b in zip(pc[:-1], pc[1:]):
                if b > a:
                    self.parts.append(index_mod.QuerySet(index, self.user_ids[a:b]))
                    self.contexts.append(_lib.Context())
                    self.streams.append(torch.cuda.Stream())

    def topk_tensors(self, k: int, work_sharing: bool = True):
        """(ids, scores, visited) of this rank's users, in ``user_ids`` order."""
        if self.queries is not None:
            return index_mod.query_batch_tensors(self.index, self.model, self.queries, k, work_sharing)
        if not self.parts:
            dev = _device.device()
            k_eff = min(k, self.model.num_items)
            return (torch.empty((0, k_eff), dtype=torch.int32, device=dev),
                    torch.empty((0, k_eff), dtype=torch.float64, device=dev),
                    torch.empty(0, dtype=torch.int64, device=dev))
        main = torch.cuda.current_stream()
        fork = torch.cuda.Event()
        fork.record(main)
        outs = []
        for q, ctx, st in zip(self.parts, self.contexts, self.streams):
            st.wait_event(fork)
            with torch.cuda.stream(st):
                outs.append(index_mod.query_batch_tensors(self.index, self.model, q, k, work_sharing,
                                                          ctx=ctx.handle))
        for st in self.streams:
            join = torch.cuda.Event()
            join.record(st)
            main.wait_event(join)
        # the parts' tensors were made on their streams: keep them alive for main's use
        for o, st in zip(outs, self.streams):
            for t in o:
                t.record_stream(main)
        return tuple(torch.cat([o[i] for o in outs]) for i in range(3))

    def stats(self):
        """(queries, continued past B, executed pairs launch 1, launch 2) summed
        over this rank's serving calls (after the stream synchronised)."""
        if not self.parts:
            nq, n_cont, _, _, _ = _lib.ws_stats()
            p1, p2 = _lib.executed_pairs()
            return nq, n_cont, p1, p2
        tot = [int(self.user_ids.size), 0, 0, 0]
        for ctx in self.contexts:
            n_cont, _, p1, p2 = ctx.stats()
            tot[1] += n_cont
            tot[2] += p1
            tot[3] += p2
        return tuple(tot)


# ---------------------------------------------------------------------------
# catalogue sharding: partial top-K per item shard + exchange + device merge
# ---------------------------------------------------------------------------

def item_shard(model: ModelPair, rank: int, world: int) -> tuple[ModelPair | None, int]:
    """All users against this rank's contiguous item shard, and its id
    offset; (None, lo) when the shard is empty (fewer items than ranks)."""
    lo, hi = shard_range(model.num_items, rank, world)
    if hi == lo:
        return None, lo
    return ModelPair(model.users, FactorMatrix(model.items.values[lo:hi])), lo


def pad_partial(ids: torch.Tensor, scores: torch.Tensor, id_offset: int, k: int):
    """A shard's partial top-K with global ids, padded to k columns with
    id -1 / score -inf (a shard may hold fewer than k items)."""
    u, kk = ids.shape
    pi = torch.full((u, k), -1, dtype=torch.int32, device=ids.device)
    ps = torch.full((u, k), float("-inf"), dtype=torch.float64, device=ids.device)
    pi[:, :kk] = torch.where(ids >= 0, ids + id_offset, ids)
    ps[:, :kk] = scores
    return pi, ps


def _host_exchange(group) -> bool:
    return dist.get_backend(group) != "nccl"


def exchange_partials(ids: torch.Tensor, scores: torch.Tensor, id_offset: int, k: int, group=None):
    """All-gather every rank's partial top-K (ids made global, padded to k
    with id -1 / -inf) -> tensors [world, U, k] on the same device."""
    world = dist.get_world_size(group)
    pi, ps = pad_partial(ids, scores, id_offset, k)
    dev = pi.device
    if _host_exchange(group):
        pi, ps = pi.cpu(), ps.cpu()
    gi = [torch.empty_like(pi) for _ in range(world)]
    gs = [torch.empty_like(ps) for _ in range(world)]
    dist.all_gather(gi, pi, group=group)
    dist.all_gather(gs, ps, group=group)
    return torch.stack(gi).to(dev), torch.stack(gs).to(dev)


def exchange_user_slices(ids: torch.Tensor, scores: torch.Tensor, id_offset: int, k: int, group=None):
    """All-to-all of partial top-K lists: rank r receives, from every rank,
    the rows of r's contiguous user slice (shard_range over the users) ->
    ([world, n_r, k] ids, [world, n_r, k] scores) on the input's device."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    nu = ids.shape[0]
    pi, ps = pad_partial(ids, scores, id_offset, k)
    dev = pi.device
    spans = [shard_range(nu, r, world) for r in range(world)]
    send = [hi - lo for lo, hi in spans]
    n_r = send[rank]
    recv = [n_r] * world
    if _host_exchange(group):
        pi, ps = pi.cpu(), ps.cpu()
    oi = torch.empty((world * n_r, k), dtype=pi.dtype, device=pi.device)
    os_ = torch.empty((world * n_r, k), dtype=ps.dtype, device=ps.device)
    dist.all_to_all_single(oi, pi, recv, send, group=group)
    dist.all_to_all_single(os_, ps, recv, send, group=group)
    return oi.view(world, n_r, k).to(dev), os_.view(world, n_r, k).to(dev)


class CatalogShard:
    """A rank's resident item shard for repeated catalogue-sharded serving."""

    def __init__(self, model: ModelPair, rank: int, world: int):
        self.model, self.lo = item_shard(model, rank, world)
        if self.model is not None:
            _device.share_rows(model.items, self.model.items, self.lo, self.lo + self.model.num_items)
        self.num_users, self.num_items = model.num_users, model.num_items
        self.users = model.users
        self.rank, self.world = rank, world
        self.user_lo, self.user_hi = shard_range(model.num_users, rank, world)

    def partial_tensors(self, k: int):
        """This shard's top-k_eff for every user, global ids, padded to k_eff."""
        k_eff = min(k, self.num_items)
        if self.model is None:
            dev = _device.f64(self.users).device
            return (torch.full((self.num_users, k_eff), -1, dtype=torch.int32, device=dev),
                    torch.full((self.num_users, k_eff), float("-inf"), dtype=torch.float64, device=dev))
        ids, sc, _ = brute.topk_matmul_tensors(self.model, k)
        return ids, sc

    def topk_tensors(self, k: int, group=None, merge=None):
        """Exact global top-K of this rank's user slice [user_lo, user_hi)."""
        k_eff = min(k, self.num_items)
        ids, sc = self.partial_tensors(k)
        off = self.lo if self.model is not None else 0
        gi, gs = exchange_user_slices(ids, sc, off, k_eff, group)
        merge = merge or _ops.merge_topk
        return merge(gi.contiguous(), gs.contiguous(), k_eff)


def catalog_sharded_topk(model: ModelPair, k: int, group=None, merge=None, exchange: str = "all_to_all"):
    """Exact global top-K with the catalogue split across the ranks of
    ``group``.  ``exchange="all_to_all"`` (default): every rank returns the
    merged lists of its own user slice, (ids int32 [n_r, k_eff], scores
    float64, first user id).  ``exchange="all_gather"``: every rank returns
    the lists of ALL users, (ids [U, k_eff], scores, 0).  ``merge`` defaults
    to the device merge kernel (simdex_merge_topk)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    shard = CatalogShard(model, rank, world)
    merge = merge or _ops.merge_topk
    k_eff = min(k, model.num_items)
    if exchange == "all_to_all":
        ids, sc = shard.topk_tensors(k, group, merge)
        return ids, sc, shard.user_lo
    if exchange != "all_gather":
        raise ValueError("exchange must be 'all_to_all' or 'all_gather'")
    ids, sc = shard.partial_tensors(k)
    gi, gs = exchange_partials(ids, sc, shard.lo if shard.model is not None else 0, k_eff, group)
    ids, sc = merge(gi.contiguous(), gs.contiguous(), k_eff)
    return ids, sc, 0


# ---------------------------------------------------------------------------
# Algorithm 2 on one rank
# ---------------------------------------------------------------------------

def run_pipeline_shard(model: ModelPair, *, k: int, rank: int, world: int, num_clusters: int = 8,
                       block_size: int = 4096, sample_fraction: float = 0.001, h0: float | None = None,
                       seed: int = 0, max_iters: int = 100, force: str | None = None, work_sharing: bool = True):
    """run_pipeline (optimizer.py:212-288) on rank ``rank`` of ``world``:
    cluster, build, estimate and decide on every rank (deterministic kernels:
    the same plan everywhere, no collective), then serve this rank's share --
    the cluster-routed users on the index branch, a contiguous user block on
    the blocked-product branch.  Returns (results of this rank's users as a
    TopKResults with global user ids, PipelineReport)."""
    from . import optimizer
    plan = optimizer.plan_pipeline(model, k=k, num_clusters=num_clusters, block_size=block_size,
                                   sample_fraction=sample_fraction, h0=h0, seed=seed, max_iters=max_iters,
                                   force=force)
    with optimizer._Stage() as t_serve:
        if plan.decision == optimizer.INDEX:
            shard = IndexShard(plan.index, model, rank, world, plan.walk)
            uids = shard.user_ids
            ids, sc, vis = shard.topk_tensors(k, work_sharing)
        else:
            shard = UserShard(model, rank, world)
            uids = np.arange(shard.lo, shard.hi, dtype=np.int64)
            ids, sc = shard.topk_tensors(k)
            vis = torch.full((ids.shape[0],), model.num_items, dtype=torch.int64, device=ids.device)
        ids_h, sc_h, vis_h = _device.to_host_pinned_many(ids, sc, vis)
        results = index_mod.TopKResults(uids, ids_h, sc_h, vis_h)
    return results, plan.report(t_serve.seconds)


def device_of(model: ModelPair):
    return _device.f64(model.users).device
