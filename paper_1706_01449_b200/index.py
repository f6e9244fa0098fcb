"""Clustered upper-bound index for exact top-K inner-product queries
(reference: mipserve/index.py).

The sorted ceiling lists live on the device (int32 item ids + float64
ceilings, [C, |I|]); the host views ``item_ids`` / ``bounds`` /
``item_norms`` of the reference's CentroidIndex are materialised on first
access.  Every query runs on the GPU: the bounded walk (simdex_walk) and the
work-sharing batch path (simdex_query_ws).  Results are exact and equal the
reference's, including ``visited``.
"""

from __future__ import annotations

import ctypes as C
import itertools
import weakref

import math
import os
import struct
from collections.abc import Mapping
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib, _ops
from .clustering import DEGENERATE_ANGLE, Clustering, angular_distance
from .model_io import DimensionMismatchError, FactorMatrix, FormatError, ModelPair, NonFiniteValueError

DEFAULT_BLOCK_SIZE = 4096

INDEX_MAGIC = b"MFIDX001"
_IDX_HEADER = struct.Struct("<8sQQQQQq")


@dataclass(frozen=True)
class TopKResult:
    """Top items for one user: scores descending, ties by ascending item id;
    ``visited`` = items whose true score was computed (index.py:42-58)."""

    user_id: int
    item_ids: np.ndarray
    scores: np.ndarray
    visited: int

    @property
    def entries(self) -> list[tuple[int, float]]:
        return list(zip(self.item_ids.tolist(), self.scores.tolist()))


class TopKResults(list):
    """``list[TopKResult]`` over batched [n, K] result arrays, built lazily.

    The reference returns a plain list (index.py:305-389, brute.py:59-113).
    This is a list subclass whose elements are created on demand: indexing,
    iteration, ``len``, ``==``, ``+`` and ``in`` work without building all n
    objects, and the first mutating call (append, sort, item assignment, ...)
    materialises every element into the list proper, after which it is an
    ordinary list.  Elements are fresh TopKResult objects with int64 / float64
    arrays, except ``reused`` positions, which return the given objects as-is
    (``precomputed`` in query_batch, index.py:330-332).  The whole-batch
    arrays are ``.item_ids`` / ``.scores`` / ``.visited`` (as computed; not
    updated by later list mutation).
    """

    def __init__(self, user_ids, item_ids, scores, visited, reused=None):
        list.__init__(self)
        # user_ids None: every user in order (position == id), materialised on request
        self._uids = None if user_ids is None else np.asarray(user_ids, dtype=np.int64)
        self._n = int(item_ids.shape[0]) if user_ids is None else int(self._uids.shape[0])
        self.item_ids = item_ids
        self.scores = scores
        self.visited = visited
        self._reused = reused or {}
        self._lazy = True

    @property
    def user_ids(self) -> np.ndarray:
        if self._uids is None:
            self._uids = np.arange(self._n, dtype=np.int64)
        return self._uids

    def _make(self, i):
        r = self._reused.get(i)
        if r is not None:
            return r
        uid = i if self._uids is None else int(self._uids[i])
        return TopKResult(uid, self.item_ids[i].astype(np.int64), self.scores[i].astype(np.float64),
                          int(self.visited[i]))

    def _materialize(self):
        if self._lazy:
            elems = [self._make(i) for i in range(self._n)]
            self._lazy = False
            list.extend(self, elems)

    # -- read access (lazy) --------------------------------------------------
    def __len__(self):
        return self._n if self._lazy else list.__len__(self)

    def __getitem__(self, i):
        if not self._lazy:
            return list.__getitem__(self, i)
        if isinstance(i, slice):
            return [self._make(j) for j in range(*i.indices(self._n))]
        i = int(i)
        if i < 0:
            i += self._n
        if not 0 <= i < self._n:
            raise IndexError("list index out of range")
        return self._make(i)

    def __iter__(self):
        if not self._lazy:
            return list.__iter__(self)
        return (self._make(i) for i in range(self._n))

    def __reversed__(self):
        if not self._lazy:
            return list.__reversed__(self)
        return (self._make(i) for i in range(self._n - 1, -1, -1))

    def __contains__(self, x):
        return any(x is e or x == e for e in self)

    def __eq__(self, other):
        if not isinstance(other, list):
            return NotImplemented
        return len(self) == len(other) and all(a is b or a == b for a, b in zip(self, other))

    def __ne__(self, other):
        eq = self.__eq__(other)
        return eq if eq is NotImplemented else not eq

    __hash__ = None

    def __add__(self, other):
        if not isinstance(other, list):
            return NotImplemented
        return list(self) + list(other)

    def __radd__(self, other):
        if not isinstance(other, list):
            return NotImplemented
        return list(other) + list(self)

    def __mul__(self, n):
        return list(self) * n

    __rmul__ = __mul__

    def __repr__(self):
        if self._lazy and self._n > 6:
            head = ", ".join(repr(self._make(i)) for i in range(3))
            return f"[{head}, ... ({self._n} results)]"
        return repr(list(self))

    def __reduce__(self):
        return (list, (list(self),))

    def copy(self):
        return list(self)

    def index(self, x, *args):
        self._materialize()
        return list.index(self, x, *args)

    def count(self, x):
        return sum(1 for e in self if e is x or e == x)

    # -- mutation: materialise, then behave as a plain list -------------------
    def _mutator(name):  # noqa: N805 -- class-body helper
        base = getattr(list, name)

        def method(self, *args, **kwargs):
            self._materialize()
            return base(self, *args, **kwargs)

        method.__name__ = name
        return method

    for _name in ("append", "extend", "insert", "pop", "remove", "clear", "sort", "reverse", "__setitem__",
                  "__delitem__", "__iadd__", "__imul__"):
        locals()[_name] = _mutator(_name)
    del _name, _mutator


class SampleResults(Mapping):
    """Read-only ``{user_id: TopKResult}`` over one batched result (the
    optimizer's sample walks, optimizer.py:141-145).  Entries are built on
    first access and kept, so every lookup -- including query_batch's reuse of
    them -- returns the same object, without a per-user host loop up front."""

    def __init__(self, results: TopKResults):
        self._res = results
        ids = results.user_ids
        self._order = None if ids.size < 2 or bool((ids[1:] > ids[:-1]).all()) else np.argsort(ids, kind="stable")
        self._sorted = ids if self._order is None else ids[self._order]
        self._cache = {}

    @property
    def user_ids(self) -> np.ndarray:
        return self._res.user_ids

    def _position(self, u):
        j = int(np.searchsorted(self._sorted, u))
        if j >= self._sorted.shape[0] or self._sorted[j] != u:
            return -1
        return j if self._order is None else int(self._order[j])

    def __getitem__(self, u):
        u = int(u)
        r = self._cache.get(u)
        if r is None:
            i = self._position(u)
            if i < 0:
                raise KeyError(u)
            r = self._cache[u] = self._res[i]
        return r

    def __contains__(self, u):
        try:
            return self._position(int(u)) >= 0
        except (TypeError, ValueError):
            return False

    def __iter__(self):
        return iter(self._res.user_ids.tolist())

    def __len__(self):
        return len(self._res)


class _Reused:
    """Positions of a query_batch answered by ``precomputed`` entries, looked
    up lazily (TopKResults only asks for the positions it materialises)."""

    def __init__(self, precomputed, uids, hit, count):
        self._pre, self._uids, self._hit, self._n = precomputed, uids, hit, count

    def get(self, i):
        if 0 <= i < self._hit.shape[0] and self._hit[i]:
            return self._pre[i if self._uids is None else int(self._uids[i])]
        return None

    def __len__(self):
        return self._n


class CentroidIndex:
    """Per-cluster item lists sorted by score ceiling, plus item norms
    (index.py:61-87).  Immutable; safe to share for reads."""

    def __init__(self, item_ids, bounds, item_norms, block_size, clustering, *, _dev=None):
        self.block_size = int(block_size)
        self.clustering = clustering
        self._host = {}
        self._dev = dict(_dev or {})
        for name, val in (("item_ids", item_ids), ("bounds", bounds), ("item_norms", item_norms)):
            if val is not None:
                a = np.asarray(val)
                a.setflags(write=False) if a.flags.owndata else None
                self._host[name] = a
        shape = self._dev["ids"].shape if "ids" in self._dev else self._host["item_ids"].shape
        self._shape = (int(shape[0]), int(shape[1]))

    # -- host views (reference fields) --------------------------------------
    def _host_get(self, name, key, dtype):
        if name not in self._host:
            a = _device.to_host(self._dev[key]).astype(dtype, copy=False)
            a.setflags(write=False)
            self._host[name] = a
        return self._host[name]

    @property
    def item_ids(self) -> np.ndarray:
        return self._host_get("item_ids", "ids", np.int64)

    @property
    def bounds(self) -> np.ndarray:
        return self._host_get("bounds", "bounds", np.float64)

    @property
    def item_norms(self) -> np.ndarray:
        return self._host_get("item_norms", "norms", np.float64)

    @property
    def num_clusters(self) -> int:
        return self._shape[0]

    @property
    def num_items(self) -> int:
        return self._shape[1]

    @property
    def entry_count(self) -> int:
        return self._shape[0] * self._shape[1]

    # -- device views -------------------------------------------------------
    def device_lists(self):
        if "ids" not in self._dev:
            self._dev["ids"] = _device.to_device(self._host["item_ids"].astype(np.int32))
            self._dev["bounds"] = _device.to_device(self._host["bounds"].astype(np.float64))
        return self._dev["ids"], self._dev["bounds"]

    def device_list_pos(self):
        """int32 [C, n]: position of each item in each cluster's list."""
        if "pos" not in self._dev:
            ids, _ = self.device_lists()
            self._dev["pos"] = _ops.list_positions(ids)
        return self._dev["pos"]

    def device_assignment(self):
        return self.clustering.device_assignment()

    def device_prefix(self, model: ModelPair, list_order: bool = False, head: int = 0):
        """Per-cluster prefix operand of ``model.items`` (cached with a strong
        reference to that matrix, so a recycled id() can never alias it).
        Default: each cluster's first B' items in its centroid's score order
        (a cluster's users meet their best items first, so their thresholds
        rise at once: ~8 % off the prefix pass at cfg2 K = 10, 10 % at K = 50);
        ``list_order``: the list (ceiling) order the prefix early exit needs,
        after the ``head`` best items by centroid score (hybrid) when head > 0."""
        head = head if list_order else 0
        key = (("prefix_hybrid", head) if head else "prefix_list") if list_order else "prefix"
        ent = self._dev.get(key)
        if ent is None or ent[0] is not model.items:
            ids, bounds = self.device_lists()
            if list_order and head:
                built = _ops.build_prefix_hybrid(_device.packed(model.items), _device.f64(model.items),
                                                 self.clustering.device_centroids(), ids, self.device_list_pos(),
                                                 bounds, self.block_size, head)
            elif list_order:
                built = _ops.build_prefix(_device.packed(model.items), ids, self.block_size)
            else:
                built = _ops.build_prefix_ordered(_device.packed(model.items), _device.f64(model.items),
                                                  self.clustering.device_centroids(), ids, self.device_list_pos(),
                                                  bounds, self.block_size)
            ent = self._dev[key] = (model.items, built)
        return ent[1]

    def device_full_lists(self, model: ModelPair):
        """Every cluster's whole list as a packed operand in list order
        (simdex_build_prefix with block = n; cached with a strong reference to
        ``model.items``): the users that go on past B scan their own cluster's
        list from B and stop on its ceilings (Algorithm 1's bound) instead of
        scanning the norm-sorted catalogue.  None when it would take more than
        FULL_LIST_BYTES (cfg4: 17.9 GB), or when the prefix is the whole list."""
        ent = self._dev.get("full_lists")
        if ent is None or ent[0] is not model.items:
            n, c = model.num_items, self.num_clusters
            pi = _device.packed(model.items)
            bf_pad = 128 * ((n + 127) // 128)
            built = None
            if min(self.block_size, n) < n and min(self.block_size, n) % 128 == 0 and \
                    c * bf_pad * pi.kp * 2 <= FULL_LIST_BYTES:
                ids, _ = self.device_lists()
                built = _ops.build_prefix(pi, ids, n)
            ent = self._dev["full_lists"] = (model.items, built)
        return ent[1]

    def device_all_users(self, num_users: int, dev):
        """(arange(num_users) on the device, its cluster grouping), cached per
        user count (a model grown by add_user gets a fresh entry)."""
        qs = self.all_users_queries(num_users, dev)
        return qs.q, qs.grouped

    def all_users_queries(self, num_users: int, dev) -> "QuerySet":
        """Every user as a QuerySet (its own execution context, so repeated
        serves skip the per-query-set setup), cached per user count."""
        key = ("all_users", int(num_users))
        ent = self._dev.get(key)
        if ent is None:
            q = torch.arange(num_users, dtype=torch.int64, device=dev)
            ent = self._dev[key] = QuerySet(self, None, q=q)
        return ent


def item_bound(item_norm: float, item_angle: float, cluster_angle: float) -> float:
    """Eq. 2 ceiling of one item (index.py:90-100): ||i|| cos(theta_ic -
    theta_b) while the slack is below the item angle, else ||i||."""
    if item_norm < 0.0:
        raise ValueError("item_norm must be >= 0")
    for name, a in (("item_angle", item_angle), ("cluster_angle", cluster_angle)):
        if not 0.0 <= a <= math.pi:
            raise ValueError(f"{name} outside [0, pi]: {a}")
    return float(item_norm * math.cos(item_angle - cluster_angle)) if cluster_angle < item_angle else float(item_norm)


def _device_build(model: ModelPair, centers_t, theta_t):
    items = _device.f64(model.items)
    return _ops.build_index(items, centers_t, theta_t)


def build_index(model: ModelPair, clustering: Clustering, block_size: int = DEFAULT_BLOCK_SIZE) -> CentroidIndex:
    """Sorted ceiling lists for every cluster, built on the GPU (index.py:129-155)."""
    if clustering.num_assigned() != model.num_users:
        raise ValueError(f"clustering covers {clustering.num_assigned()} users, model has {model.num_users}")
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    norms, ids, bounds = _device_build(model, clustering.device_centroids(), clustering.device_max_angle())
    index = CentroidIndex(None, None, None, block_size, clustering, _dev={"ids": ids, "bounds": bounds, "norms": norms})
    # the inverse list positions (visited in closed form) are part of the
    # build; the prefix operand is built by prepare_serving / the first
    # work-sharing query, in the layout the walk estimate selects (building the
    # default layout here cost run_pipeline 0.5 ms for an operand it replaced)
    index.device_list_pos()
    return index


def _check_k(k):
    if k < 1:
        raise ValueError("k must be >= 1")


def _walk_rows(index, model, q_users_np, k, q_clusters=None):
    users = _device.f64(model.users)
    unorm = _device.norms(model.users)
    items = _device.f64(model.items)
    ids, bounds = index.device_lists()
    q = _device.to_device(np.asarray(q_users_np, dtype=np.int64))
    if q_clusters is None:
        qc = index.device_assignment().index_select(0, q).to(torch.int32)
    else:
        qc = q_clusters
    return _ops.walk(users, unorm, items, ids, bounds, q, qc, k, users32=_device.f32_exact(model.users),
                     items32=_device.f32_exact(model.items))


def query_user(index: CentroidIndex, model: ModelPair, user_id: int, k: int) -> TopKResult:
    """Exact top-K for one model user via their cluster's list walk (index.py:258-268)."""
    _check_k(k)
    if not 0 <= user_id < model.num_users:
        raise ValueError(f"user_id {user_id} out of range [0, {model.num_users})")
    ids, sc, vis = _walk_rows(index, model, [user_id], k)
    return TopKResult(int(user_id), _device.to_host(ids[0]).astype(np.int64), _device.to_host(sc[0]),
                      int(vis[0].item()))


def _check_vector(vector, factors: int, what="vector") -> np.ndarray:
    v = np.asarray(vector, dtype=np.float64)
    if v.shape != (factors,):
        raise DimensionMismatchError(f"{what} shape {v.shape} != ({factors},)")
    if not np.isfinite(v).all():
        raise NonFiniteValueError(f"{what} contains non-finite values")
    return v


def _nearest_centroid(cvals: np.ndarray, v: np.ndarray):
    """Route a vector to its L2-nearest centroid and measure its angle
    (index.py:285-293); host-side scalar routing, like the reference."""
    c = int(((cvals - v) ** 2).sum(axis=1).argmin())
    if np.linalg.norm(v) == 0.0 or np.linalg.norm(cvals[c]) == 0.0:
        return c, DEGENERATE_ANGLE
    return c, angular_distance(v, cvals[c])


def _cluster_list(model, centroid, slack):
    """One re-bounded list (index.py:295-299): GPU build for a single centroid."""
    dev = _device.device()
    cen = torch.as_tensor(np.asarray(centroid, dtype=np.float64)[None, :], device=dev)
    th = torch.tensor([float(slack)], dtype=torch.float64, device=dev)
    _, ids, bounds = _device_build(model, cen, th)
    return ids, bounds


def query_vector(index: CentroidIndex, model: ModelPair, vector, k: int) -> TopKResult:
    """Exact top-K for an arbitrary query vector (user_id -1); a vector outside
    its cluster's recorded slack walks a locally re-bounded list (index.py:271-302)."""
    _check_k(k)
    u = _check_vector(vector, model.factors, "vector")
    cvals = index.clustering.centroids.values
    c, theta = _nearest_centroid(cvals, u)
    dev = _device.device()
    ut = torch.as_tensor(u[None, :], device=dev)
    un = torch.tensor([float(np.linalg.norm(u))], dtype=torch.float64, device=dev)
    if theta <= index.clustering.max_angle[c]:
        ids, bounds = index.device_lists()
        qc = torch.tensor([c], dtype=torch.int32, device=dev)
    else:
        ids, bounds = _cluster_list(model, cvals[c], theta)
        qc = torch.zeros(1, dtype=torch.int32, device=dev)
    q = torch.zeros(1, dtype=torch.int64, device=dev)
    u32 = u.astype(np.float32)
    ut32 = torch.as_tensor(u32[None, :], device=dev) if np.array_equal(u32.astype(np.float64), u) else None
    oi, os_, ov = _ops.walk(ut, un, _device.f64(model.items), ids, bounds, q, qc, k, users32=ut32,
                            items32=_device.f32_exact(model.items))
    return TopKResult(-1, _device.to_host(oi[0]).astype(np.int64), _device.to_host(os_[0]), int(ov[0].item()))


# The prefix pass of work sharing ends a 128-query unit early (every query's
# certified K-th above ||u|| x the list ceiling of the next tile) when the
# optimizer's walk estimate for this index and K says walks are short against
# B: below this fraction of B' the exit saves more tensor work than its
# bookkeeping costs (tools/exit_ab.py, all-user serve: cfg4 K=10, mean walk
# 47 of 4,096, 2.95 -> 2.10 ms; cfg2 K=5, walk 0.30 B', 0.97 -> 0.95 ms;
# cfg2 K=10, walk 0.44 B', break-even; cfg2 K=50, walk B', +2 %).
# Round 2: between PREFIX_LIST_FRACTION and PREFIX_EXIT_FRACTION the prefix is
# laid out "hybrid" -- its PREFIX_HEAD (128) best items by centroid score first (the
# thresholds rise at once), the rest in list order (the exit can end a warp
# inside the prefix): cfg2 K=10 gemm 0.457 -> 0.402 ms, K=5 0.390 -> 0.300
# (tools/ab_run_hybrid.sh); below PREFIX_LIST_FRACTION (cfg4: walks of 0.015
# B') the pure list order stays faster (0.479 vs 0.584 ms).
PREFIX_EXIT_FRACTION = 0.6
PREFIX_LIST_FRACTION = 0.1


def note_walk_estimate(index: CentroidIndex, k: int, mean_visited: float) -> None:
    index._dev[("walk_estimate", int(k))] = float(mean_visited)


def prepare_serving(index: CentroidIndex, model: ModelPair, k: int) -> None:
    """Build the prefix operand the next work-sharing query at depth ``k``
    will use (the order follows the early-exit decision), so a timed serve
    does not build it."""
    if model.factors <= 256 and min(k, model.num_items) <= 256:
        opts = _ws_options(index, k, model.num_items, True)
        index.device_prefix(model, list_order=bool(opts & _ops.WS_PREFIX_EXIT),
                            head=_prefix_head(index, k, model.num_items))


def _ws_options(index: CentroidIndex, k: int, n: int, work_sharing: bool) -> int:
    mv = index._dev.get(("walk_estimate", int(k)))
    if not work_sharing or mv is None:
        return 0
    return _ops.WS_PREFIX_EXIT if mv < PREFIX_EXIT_FRACTION * min(index.block_size, n) else 0


def _prefix_head(index: CentroidIndex, k: int, n: int) -> int:
    """Head of the hybrid prefix layout for the exit (0: pure list order)."""
    mv = index._dev.get(("walk_estimate", int(k)))
    if mv is None or mv < PREFIX_LIST_FRACTION * min(index.block_size, n):
        return 0
    return PREFIX_HEAD


# the list-order catalogue pass (csrc/gemm_topk.cu: SIMDEX_LIST_MIN_K,
# SIMDEX_LIST_MIN_Q) serves query sets of 50k users or more from K = 8 on; its
# per-cluster full-list operand (0.8 ms, 583 MB at cfg2) is built once an
# index has served FULL_LISTS_AFTER such batches -- a one-shot run_pipeline
# saves 0.11 ms per serve with it and would pay 0.8 ms to build it
LIST_MIN_K, LIST_MIN_Q = 8, 50000
FULL_LISTS_AFTER = int(os.environ.get("SIMDEX_FULL_LISTS_AFTER", "1"))


def _full_lists_for(index: CentroidIndex, model: ModelPair, k: int, nq: int):
    ent = index._dev.get("full_lists")
    if ent is not None and ent[0] is model.items:
        return ent[1]
    if min(k, model.num_items) < LIST_MIN_K or nq < LIST_MIN_Q:
        return None
    served = index._dev.get("list_pass_serves", 0)
    index._dev["list_pass_serves"] = served + 1
    return index.device_full_lists(model) if served >= FULL_LISTS_AFTER else None


_QUERY_TOKENS = itertools.count(1)
# the hybrid prefix's head (see PREFIX_EXIT_FRACTION)
PREFIX_HEAD = int(os.environ.get("SIMDEX_PREFIX_HEAD", "128"))
# largest per-cluster full-list operand built for the list-order catalogue pass
FULL_LIST_BYTES = int(os.environ.get("SIMDEX_FULL_LIST_BYTES", str(4 << 30)))


class QuerySet:
    """A fixed set of user rows prepared for repeated serving on one index:
    the device id tensor and its grouping by cluster (simdex_group_queries),
    computed once, and a token unique to this object
    (simdex_ctx_set_query_token): a serve that finds this set's setup still
    in its execution context's workspace (no other call in between) skips
    the per-query-set setup kernels (units, packed query rows, norms).  Used
    by the all-users serve and the multi-GPU shards."""

    def __init__(self, index: CentroidIndex, user_ids, q=None):
        # weak: the index caches its all-users set, and a reference cycle would
        # keep a dropped index's device tensors (lists, operands) alive until
        # the cyclic collector runs -- every rebuild would then cudaMalloc anew
        self._index = weakref.ref(index)
        if q is None:
            ids = np.asarray(user_ids, dtype=np.int64)
            self.user_ids = ids
            self.q = _device.to_device(ids)
        else:
            self.user_ids = None if user_ids is None else np.asarray(user_ids, dtype=np.int64)
            self.q = q
        self.grouped = _ops.group_queries(self.q, index.device_assignment(), index.num_clusters)
        self.token = next(_QUERY_TOKENS)
        self._serves = 0
        self._own_ctx = None

    @property
    def index(self):
        return self._index()

    def serving_context(self):
        """The execution context this set is served on when the caller names
        none: the thread's default for its first serve (a one-shot pipeline
        allocates nothing), its own from the second serve on -- nothing else
        then disturbs the setup the set keeps in that context's workspace
        (which a CUDA graph captured from a serve relies on), and the arena
        is allocated once at its final size."""
        self._serves += 1
        if self._serves >= 2 and self._own_ctx is None:
            self._own_ctx = _lib.Context()
        return None if self._own_ctx is None else self._own_ctx.handle

    def context(self, ctx=None):
        """Tag the context the next serve runs on (``ctx``, or None for the
        thread's default) with this set's token; returns ``ctx``."""
        _lib.call("simdex_ctx_set_query_token", ctx, C.c_int64(self.token))
        return ctx

    def __len__(self):
        return int(self.q.shape[0])


def query_batch_tensors(index: CentroidIndex, model: ModelPair, q_users, k: int, work_sharing: bool = True,
                        ctx=None):
    """Device form of query_batch: int64 user rows in (a device tensor, a
    QuerySet of this index, or None for every user), (ids int32 [n, k_eff],
    scores float64, visited int64) out, all on the device, in query order."""
    users = _device.f64(model.users)
    items = _device.f64(model.items)
    ids, bounds = index.device_lists()
    n = model.num_items
    grouped = None
    qs = None
    if q_users is None:
        qs = index.all_users_queries(model.num_users, users.device)
        if ctx is None:
            ctx = qs.serving_context()
    elif isinstance(q_users, QuerySet):
        if q_users.index is not index:
            raise ValueError("QuerySet was prepared for another index")
        qs = q_users
    if qs is not None:
        q_users, grouped = qs.q, qs.grouped
    pu, pi = _device.packed_users(model.users), _device.packed_sorted(model.items)
    if min(k, n) <= 256 and pu.kp <= 256:
        # tensor-core path; without work sharing every query takes the full-list
        # pass (block 0) and visited is Algorithm 1's stop position, exactly the walk's
        if grouped is None:
            grouped = _ops.group_queries(q_users, index.device_assignment(), index.num_clusters)
        block = index.block_size if work_sharing else 0
        options = _ws_options(index, k, n, work_sharing)
        prefix = (index.device_prefix(model, list_order=bool(options & _ops.WS_PREFIX_EXIT),
                                      head=_prefix_head(index, k, n)) if work_sharing else (None, None, 0))
        if qs is not None:
            ctx = qs.context(ctx)
        if work_sharing and block < n:
            fl = _full_lists_for(index, model, k, int(q_users.shape[0]))
            if fl is not None:
                _lib.call("simdex_ctx_set_full_lists", ctx, _lib.ptr(fl[0]), _lib.ptr(fl[1]), fl[2])
        return _ops.query_ws(users, pu, items, pi, ids, index.device_list_pos(), bounds, block, prefix, grouped, k,
                             items32=_device.f32_exact(model.items), users32=_device.f32_exact(model.users),
                             options=options, ctx=ctx)
    qc = index.device_assignment().index_select(0, q_users).to(torch.int32)
    out = _ops.walk(users, _device.norms(model.users), items, ids, bounds, q_users, qc, k,
                    users32=_device.f32_exact(model.users), items32=_device.f32_exact(model.items))
    if work_sharing:  # k beyond the tensor-core envelope: WS visited = n if B >= n else max(B, walk visited)
        vis = out[2].fill_(n) if index.block_size >= n else out[2].clamp_(min=index.block_size)
        out = (out[0], out[1], vis)
    return out


# Serving every user and returning the results to the host: the users are cut
# into contiguous id ranges served one after the other, each range's results
# copied to pinned host memory on a side stream while the next range is
# served (58 MB of results take 1.2 ms over PCIe against a 0.95 ms serve at
# cfg2).  Ranges keep 100k users or more so that each still takes the
# list-order catalogue pass.
D2H_PARTS = int(os.environ.get("SIMDEX_D2H_PARTS", "2"))
D2H_MIN_USERS_PER_PART = 100_000


def _d2h_parts(model: ModelPair, k: int) -> int:
    if min(k, model.num_items) > 256 or model.factors > 256:
        return 1
    return max(1, min(D2H_PARTS, model.num_users // D2H_MIN_USERS_PER_PART))


def _serve_all_users_overlapped(index: CentroidIndex, model: ModelPair, k: int, work_sharing: bool, parts: int):
    """query_batch_tensors over ``parts`` contiguous user ranges (cached
    QuerySets, each with its own execution context so their setups stay
    reusable), device -> pinned host copies of a range overlapped with the
    next range's kernels.  Returns host (ids, scores, visited) in user order."""
    n, k_eff = model.num_users, min(k, model.num_items)
    dev = _device.f64(model.users).device
    key = ("user_ranges", n, parts)
    ranges = index._dev.get(key)
    if ranges is None:
        cuts = [n * i // parts for i in range(parts + 1)]
        ranges = index._dev[key] = [
            (lo, hi, QuerySet(index, None, q=torch.arange(lo, hi, dtype=torch.int64, device=dev)), _lib.Context())
            for lo, hi in zip(cuts[:-1], cuts[1:])]
    ids_h = torch.empty((n, k_eff), dtype=torch.int32, pin_memory=True)
    sc_h = torch.empty((n, k_eff), dtype=torch.float64, pin_memory=True)
    vis_h = torch.empty(n, dtype=torch.int64, pin_memory=True)
    main = torch.cuda.current_stream()
    side = _device.side_stream(dev)
    for lo, hi, qs, ctx in ranges:
        ids, sc, vis = query_batch_tensors(index, model, qs, k, work_sharing, ctx=ctx.handle)
        served = torch.cuda.Event()
        served.record(main)
        with torch.cuda.stream(side):
            side.wait_event(served)
            ids_h[lo:hi].copy_(ids, non_blocking=True)
            sc_h[lo:hi].copy_(sc, non_blocking=True)
            vis_h[lo:hi].copy_(vis, non_blocking=True)
        for t in (ids, sc, vis):
            t.record_stream(side)
    side.synchronize()
    return ids_h.numpy(), sc_h.numpy(), vis_h.numpy()


def query_batch(index: CentroidIndex, model: ModelPair, user_ids=None, k: int = 1, work_sharing: bool = True,
                precomputed: dict | None = None) -> TopKResults:
    """Top-K for many users (index.py:305-389); identical entries with work
    sharing on or off.  With work sharing the first ``block_size`` items of
    each cluster's list are scored for all that cluster's users as one
    tensor-core product, and only users whose K-th does not beat the ceiling
    at B continue walking.  ``precomputed`` results are reused verbatim."""
    _check_k(k)
    all_users = user_ids is None
    n_q = model.num_users
    uids = None  # all users: positions are the ids
    if not all_users:
        uids = np.asarray([int(u) for u in user_ids], dtype=np.int64)
        bad = (uids < 0) | (uids >= model.num_users)
        if bad.any():
            raise ValueError(f"user_id {int(uids[np.argmax(bad)])} out of range [0, {model.num_users})")
        n_q = uids.shape[0]
    reused = {}
    hit = None
    if precomputed:
        if isinstance(precomputed, SampleResults):
            keys = precomputed.user_ids
        else:
            keys = np.fromiter(precomputed.keys(), dtype=np.int64, count=len(precomputed))
        keys = keys[(keys >= 0) & (keys < model.num_users)]
        mark = np.zeros(model.num_users, dtype=bool)  # O(U) membership instead of a sort-based isin
        mark[keys] = True
        hit = mark if all_users else mark[uids]
        reused = _Reused(precomputed, uids, hit, int(np.count_nonzero(hit)))
    k_eff = min(k, model.num_items)
    if len(reused) * 2 <= n_q:
        # few reused entries: serve every position on the device (the reused
        # positions still return the precomputed objects), no host gather
        if all_users and _d2h_parts(model, k) > 1:
            # from an index's second all-user serve on (the ranges' query sets
            # and contexts are one-time costs a one-shot run_pipeline would only pay)
            served = index._dev.get("all_user_serves", 0)
            index._dev["all_user_serves"] = served + 1
            if served >= 1:
                ids_h, sc_h, vis_h = _serve_all_users_overlapped(index, model, k, work_sharing,
                                                                 _d2h_parts(model, k))
                return TopKResults(uids, ids_h, sc_h, vis_h, reused)
        q = None if all_users else _device.to_device(uids)
        ids, sc, vis = query_batch_tensors(index, model, q, k, work_sharing)
        ids_h, sc_h, vis_h = _device.to_host_pinned_many(ids, sc, vis)
        return TopKResults(uids, ids_h, sc_h, vis_h, reused)
    todo = np.flatnonzero(~hit)
    ids_h = np.zeros((n_q, k_eff), dtype=np.int32)
    sc_h = np.zeros((n_q, k_eff), dtype=np.float64)
    vis_h = np.zeros(n_q, dtype=np.int64)
    if todo.size:
        ids, sc, vis = query_batch_tensors(index, model, _device.to_device(todo if all_users else uids[todo]), k,
                                           work_sharing)
        ids_h[todo] = _device.to_host(ids)
        sc_h[todo] = _device.to_host(sc)
        vis_h[todo] = _device.to_host(vis)
    return TopKResults(uids, ids_h, sc_h, vis_h, reused)


def insert_item(index: CentroidIndex, model: ModelPair, item_vector):
    """Add one item (index.py:401-430).  The lists are rebuilt on the GPU with
    the unchanged clustering: the new id is the largest, so among equal
    ceilings it sorts last -- the same list the reference's searchsorted
    insertion produces.  Returns (index, model)."""
    v = _check_vector(item_vector, model.factors, "vector")
    new_model = ModelPair(model.users, FactorMatrix(np.vstack([model.items.values, v[None, :]])))
    cl = index.clustering
    norms, ids, bounds = _device_build(new_model, cl.device_centroids(), cl.device_max_angle())
    return CentroidIndex(None, None, None, index.block_size, cl,
                         _dev={"ids": ids, "bounds": bounds, "norms": norms}), new_model


def add_user(index: CentroidIndex, model: ModelPair, user_vector):
    """Assign a new user to the L2-nearest centroid (index.py:433-483); if its
    angle exceeds the cluster's slack the slack is raised and that cluster's
    list rebuilt (flag False = drift).  Returns (index, model, fits)."""
    v = _check_vector(user_vector, model.factors, "vector")
    cl = index.clustering
    cvals = cl.centroids.values
    c, theta = _nearest_centroid(cvals, v)
    new_id = model.num_users
    new_model = ModelPair(FactorMatrix(np.vstack([model.users.values, v[None, :]])), model.items)
    assignment = np.append(cl.assignment, np.int64(c))
    members = tuple(np.append(m, new_id) if j == c else m for j, m in enumerate(cl.members))
    fits = bool(theta <= cl.max_angle[c])
    max_angle = cl.max_angle.copy()
    if not fits:
        max_angle[c] = theta
    max_angle.setflags(write=False)
    assignment.setflags(write=False)
    new_cl = Clustering(cl.centroids, assignment, max_angle, members, cl.objective, cl.seed)
    if fits:
        return _derive(index, new_cl), new_model, True
    ids, bounds = index.device_lists()
    ids, bounds = ids.clone(), bounds.clone()
    rid, rb = _cluster_list(model, cvals[c], theta)
    ids[c] = rid[0]
    bounds[c] = rb[0]
    return _derive(index, new_cl, (ids, bounds)), new_model, False


def _derive(index: CentroidIndex, clustering: Clustering, lists=None) -> CentroidIndex:
    """Same lists (or replaced ``lists``) under a new clustering."""
    out = CentroidIndex.__new__(CentroidIndex)
    out.block_size = index.block_size
    out.clustering = clustering
    out._shape = index._shape
    out._host = dict(index._host)
    # the user grouping depends on the clustering (always new here); the
    # prefix operand and list positions on the lists; walk estimates stay
    # (they only pick an option, the results are identical either way)
    out._dev = {key: val for key, val in index._dev.items()
                if not (isinstance(key, tuple) and key[0] in ("all_users", "user_ranges"))}
    if lists is not None:
        out._host.pop("item_ids", None)
        out._host.pop("bounds", None)
        out._dev["ids"], out._dev["bounds"] = lists
        out._dev.pop("pos", None)
        out._dev.pop("prefix", None)
        out._dev.pop("prefix_list", None)
        for key in [key for key in out._dev if isinstance(key, tuple) and key[0] == "prefix_hybrid"]:
            out._dev.pop(key)
        out._dev.pop("full_lists", None)
    return out


def save_index(index: CentroidIndex, path) -> None:
    """MFIDX001 sidecar (index.py:486-509): header, theta_b, centroids,
    assignment, item norms, item ids (int64), ceilings (float64)."""
    cl = index.clustering
    parts = [
        _IDX_HEADER.pack(INDEX_MAGIC, index.num_clusters, index.num_items, cl.centroids.factors,
                         cl.assignment.shape[0], index.block_size, cl.seed),
        np.ascontiguousarray(cl.max_angle, dtype="<f8").tobytes(),
        np.ascontiguousarray(cl.centroids.values, dtype="<f8").tobytes(),
        np.ascontiguousarray(cl.assignment, dtype="<i8").tobytes(),
        np.ascontiguousarray(index.item_norms, dtype="<f8").tobytes(),
        np.ascontiguousarray(index.item_ids, dtype="<i8").tobytes(),
        np.ascontiguousarray(index.bounds, dtype="<f8").tobytes(),
    ]
    with open(path, "wb") as fh:
        fh.writelines(parts)


def load_index(path) -> CentroidIndex:
    """Read a sidecar written by save_index (index.py:512-553)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _IDX_HEADER.size:
        raise FormatError(f"{path}: file shorter than the index header")
    magic, nc, n, f, nu, block, seed = _IDX_HEADER.unpack_from(raw)
    if magic != INDEX_MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}, expected {INDEX_MAGIC!r}")
    counts = [nc, nc * f, nu, n, nc * n, nc * n]
    if len(raw) != _IDX_HEADER.size + 8 * sum(counts):
        raise FormatError(f"{path}: file is {len(raw)} bytes, expected {_IDX_HEADER.size + 8 * sum(counts)}")
    off = _IDX_HEADER.size
    out = []
    for cnt, dt in zip(counts, ("<f8", "<f8", "<i8", "<f8", "<i8", "<f8")):
        out.append(np.frombuffer(raw, dtype=dt, count=cnt, offset=off).copy())
        off += 8 * cnt
    max_angle, cen, assign, norms, ids, bounds = out
    for a in (assign, max_angle):
        a.setflags(write=False)
    members = tuple(np.flatnonzero(assign == c) for c in range(nc))
    cl = Clustering(FactorMatrix(cen.reshape(nc, f)), assign, max_angle, members, np.empty(0), int(seed))
    return CentroidIndex(ids.reshape(nc, n), bounds.reshape(nc, n), norms, int(block), cl)
