"""Brute-force top-K serving (reference: mipserve/brute.py).

``topk_matmul`` runs the users x items product on tcgen05 tensor cores with
the running top-K fused into the epilogue and exact float64 rescoring of the
certified candidates (simdex_topk_matmul); ``topk_naive`` is the exact
float64 full scan + ordering on the GPU (simdex_topk_exact).  Both return
identical results under the shared tie rule (score desc, item id asc).
"""

from __future__ import annotations

import sys
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _ops
from .index import TopKResults
from .model_io import FactorMatrix, ModelPair

# tiles the reference's default_blocks picks (brute.py:21-40); accepted for
# API compatibility, the GPU tiling is internal
_TILE_BUDGET_DOUBLES = 32768
MATMUL_MAX_K = 256


@dataclass(frozen=True)
class BlockSpec:
    user_block: int
    item_block: int

    def __post_init__(self):
        if self.user_block < 1 or self.item_block < 1:
            raise ValueError("block sizes must be >= 1")


def default_blocks(factors: int) -> BlockSpec:
    """Largest power-of-two square tile whose two panels plus score tile fit
    32768 doubles (brute.py:36-40)."""
    side = 256
    while side > 8 and 2 * side * factors + side * side > _TILE_BUDGET_DOUBLES:
        side //= 2
    return BlockSpec(side, side)


def _results(ids, sc, n_items, num_users):
    vis = np.full(num_users, n_items, dtype=np.int64)
    ids_h, sc_h = _device.to_host_pinned_many(ids, sc)
    return TopKResults(None, ids_h, sc_h, vis)  # every user, in order


def topk_naive_tensors(model: ModelPair, k: int):
    return _ops.topk_exact(_device.f64(model.users), _device.f64(model.items), k)


def topk_naive(model: ModelPair, k: int) -> TopKResults:
    """Score every pair in float64 and order (brute.py:43-56); GPU exact scan."""
    if k < 1:
        raise ValueError("k must be >= 1")
    ids, sc = topk_naive_tensors(model, k)
    return _results(ids, sc, model.num_items, model.num_users)


def topk_matmul_tensors(model: ModelPair, k: int, heap_ops: bool = False, ctx=None):
    """Device form: (ids int32 [U, k_eff], scores float64, heap_ops|None);
    ``ctx``: an execution context of the caller's (_lib.Context().handle)."""
    users, items = _device.f64(model.users), _device.f64(model.items)
    if min(k, model.num_items) > MATMUL_MAX_K:
        ids, sc = _ops.topk_exact(users, items, k)
        return ids, sc, None
    return _ops.topk_matmul(users, _device.packed_users(model.users), items, _device.packed_sorted(model.items), k,
                            heap_ops, items32=_device.f32_exact(model.items), users32=_device.f32_exact(model.users),
                            ctx=ctx)


def topk_matmul(model: ModelPair, k: int, blocks: BlockSpec | None = None, counters: dict | None = None) -> TopKResults:
    """Blocked product with a running per-user top-K; identical to topk_naive
    (brute.py:59-113).  ``counters['heap_ops']`` receives per-user counts of
    tile scores that beat the running K-th when merged."""
    if k < 1:
        raise ValueError("k must be >= 1")
    ids, sc, hops = topk_matmul_tensors(model, k, heap_ops=counters is not None)
    if counters is not None:
        counters["heap_ops"] = _device.to_host(hops) if hops is not None else np.full(
            model.num_users, model.num_items, dtype=np.int64)
    return _results(ids, sc, model.num_items, model.num_users)


def _scan_list(model: ModelPair):
    """Identity list (all items in id order) for the unpruned per-pair scan."""
    cache = model.items.__dict__.setdefault("_device", {}).setdefault(_device.device().index, {})
    if "scan_list" not in cache:
        n = model.num_items
        dev = _device.device()
        cache["scan_list"] = (torch.arange(n, dtype=torch.int32, device=dev).view(1, n),
                              torch.full((1, n), float("inf"), dtype=torch.float64, device=dev))
    return cache["scan_list"]


def _perpair_scan(model: ModelPair, k: int) -> None:
    """Pair-at-a-time scoring with a bounded running top-K and no pruning
    (brute.py:116-130): the bounded-walk kernel over an unpruned list, the
    GPU's "unblocked" rate for calibrating h0."""
    ids, bounds = _scan_list(model)
    dev = _device.device()
    q = torch.arange(model.num_users, dtype=torch.int64, device=dev)
    qc = torch.zeros(model.num_users, dtype=torch.int32, device=dev)
    _ops.walk(_device.f64(model.users), _device.norms(model.users), _device.f64(model.items), ids, bounds, q, qc,
              k, no_prune=True, users32=_device.f32_exact(model.users), items32=_device.f32_exact(model.items))


@dataclass(frozen=True)
class ThroughputSample:
    """Scored pairs per second for the blocked product and the per-pair loop."""

    blocked_rate: float
    unblocked_rate: float


# GPU throughput is a saturation figure: a model smaller than this many
# (user, item) pairs is measured with its users tiled up to it (the rate per
# pair of a launch-bound run would measure launch latency, not the hardware
# factor h0 stands for, optimizer.py:69-102).
CALIBRATION_PAIRS = 1 << 28


def _calibration_model(model: ModelPair) -> ModelPair:
    pairs = model.num_users * model.num_items
    if pairs >= CALIBRATION_PAIRS:
        return model
    cache = model.users.__dict__.setdefault("_calibration", {})
    key = id(model.items)
    ent = cache.get(key)
    if ent is None or ent[0] is not model.items:
        reps = -(-CALIBRATION_PAIRS // pairs)
        reps = max(1, min(reps, (1 << 22) // model.num_users))  # at most ~4M users
        ent = cache[key] = (model.items, ModelPair(FactorMatrix(np.tile(model.users.values, (reps, 1))), model.items))
    return ent[1]


def measure_throughput(model: ModelPair, k: int = 1, blocks: BlockSpec | None = None) -> ThroughputSample:
    """Scored pairs per second of both serving styles (brute.py:141-150): the
    tensor-core blocked product and the per-pair scan, each timed warm
    (operands packed, workspace grown) with device synchronisation, on the
    model -- or, below CALIBRATION_PAIRS, its users tiled up to that size."""
    m = _calibration_model(model)
    pairs = m.num_users * m.num_items
    # module-attribute lookups at call time, like the reference (its tests
    # monkeypatch brute.topk_matmul / _perpair_scan)
    mod = sys.modules[__name__]
    mod.topk_matmul(m, k, blocks)
    mod._perpair_scan(m, k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    mod.topk_matmul(m, k, blocks)
    torch.cuda.synchronize()
    blocked = max(time.perf_counter() - t0, 1e-9)
    t0 = time.perf_counter()
    mod._perpair_scan(m, k)
    torch.cuda.synchronize()
    unblocked = max(time.perf_counter() - t0, 1e-9)
    return ThroughputSample(pairs / blocked, pairs / unblocked)
