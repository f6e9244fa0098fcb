"""Multi-GPU sharding of the serving path.

* User sharding (configs 1-4): ranks serve disjoint user ranges with the
  whole catalogue and index resident; no data-path collective.
* Catalogue sharding (config 5, 1M x 1M): every rank scores ALL users
  against its contiguous item shard (certified tensor-core top-K), the
  per-rank partial [U, K] lists are all-gathered (NCCL over NVLink on B200)
  and merged on the device by (score desc, global id asc)
  (simdex_merge_topk).  Merging the per-shard exact top-K lists gives the
  global exact top-K: every global top-K item is in its own shard's top-K.

One process per GPU, ``torch.distributed`` for the plumbing.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _device, _ops, brute
from .model_io import FactorMatrix, ModelPair


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of ``n`` rows for ``rank``."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def user_shard(model: ModelPair, rank: int, world: int) -> tuple[ModelPair, int]:
    """This rank's users (whole catalogue) and the global id of its first user."""
    lo, hi = shard_range(model.num_users, rank, world)
    return ModelPair(FactorMatrix(model.users.values[lo:hi]), model.items), lo


def item_shard(model: ModelPair, rank: int, world: int) -> tuple[ModelPair, int]:
    """All users against this rank's contiguous item shard, and its id offset."""
    lo, hi = shard_range(model.num_items, rank, world)
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


def exchange_partials(ids: torch.Tensor, scores: torch.Tensor, id_offset: int, k: int, group=None):
    """All-gather every rank's partial top-K (ids made global, padded to k
    with id -1 / -inf) -> tensors [world, U, k] on the same device."""
    world = dist.get_world_size(group)
    pi, ps = pad_partial(ids, scores, id_offset, k)
    gi = [torch.empty_like(pi) for _ in range(world)]
    gs = [torch.empty_like(ps) for _ in range(world)]
    dist.all_gather(gi, pi, group=group)
    dist.all_gather(gs, ps, group=group)
    return torch.stack(gi), torch.stack(gs)


def catalog_sharded_topk(model: ModelPair, k: int, group=None, merge=None):
    """Exact global top-K with the catalogue split across the ranks of
    ``group``.  Returns (ids int32 [U, k_eff], scores float64) on every rank.
    ``merge`` defaults to the device merge kernel (simdex_merge_topk)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    part, off = item_shard(model, rank, world)
    k_eff = min(k, model.num_items)
    ids, sc, _ = brute.topk_matmul_tensors(part, k)
    gi, gs = exchange_partials(ids, sc, off, k_eff, group)
    merge = merge or _ops.merge_topk
    return merge(gi.contiguous(), gs.contiguous(), k_eff)


def user_sharded_topk(model: ModelPair, k: int, group=None):
    """Exact top-K of this rank's users (no collective); returns (ids, scores, first user id)."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    part, lo = user_shard(model, rank, world)
    ids, sc, _ = brute.topk_matmul_tensors(part, k)
    return ids, sc, lo


def device_of(model: ModelPair):
    return _device.f64(model.users).device
