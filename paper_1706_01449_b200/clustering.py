"""k-means over user vectors plus the per-cluster angular slack theta_b
(reference: mipserve/clustering.py).

Lloyd iterations run on the GPU: k-means++ seeding with the reference's
exact RNG draw sequence (simdex_kmeans_seed), fused distance + argmin
assignment (simdex_kmeans_assign), deterministic centroid means
(simdex_kmeans_update) and theta_b (simdex_max_angles).  The host only
drives the loop: one small device->host read per iteration for the
convergence test and the empty-cluster check.
"""

from __future__ import annotations

import itertools
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _ops
from .model_io import FactorMatrix

DEFAULT_NUM_CLUSTERS = 8
DEFAULT_MAX_ITERS = 100
_LLOYD_BATCH = 3  # Lloyd iterations queued per host read (see kmeans)

# Angle used when a vector has zero norm; the most conservative choice
# (clustering.py:21-23).
DEGENERATE_ANGLE = math.pi


_RUN_TOKENS = itertools.count(1)


@dataclass(frozen=True, eq=False)
class Clustering:
    """Centroids, assignment, theta_b (``max_angle``), members, objective
    history and seed (clustering.py:26-44)."""

    centroids: FactorMatrix
    assignment: np.ndarray
    max_angle: np.ndarray
    members: tuple
    objective: np.ndarray
    seed: int

    @property
    def num_clusters(self) -> int:
        return self.centroids.rows

    # device copies (cached per device)
    def _dev(self):
        store = self.__dict__.setdefault("_device_cache", {})
        return store.setdefault(_device.device().index, {})

    def device_assignment(self) -> torch.Tensor:
        d = self._dev()
        if "assign" not in d:
            d["assign"] = _device.to_device(np.asarray(self.assignment, dtype=np.int64))
        return d["assign"]

    def device_centroids(self) -> torch.Tensor:
        return _device.f64(self.centroids)

    def device_max_angle(self) -> torch.Tensor:
        d = self._dev()
        if "theta" not in d:
            d["theta"] = _device.to_device(np.asarray(self.max_angle, dtype=np.float64))
        return d["theta"]

    def num_assigned(self) -> int:
        return int(self.assignment.shape[0])


class _DeviceClustering(Clustering):
    """What kmeans() returns: centroids, theta_b and the objective history
    are read back at once (a few values per cluster); the per-user assignment
    and the member lists stay on the device until first read on the host
    (the pipeline's build and serve use the device copies only)."""

    def __init__(self, centroids, max_angle, objective, seed, assign_dev, members_dev, offsets):
        for name, val in (("centroids", centroids), ("max_angle", max_angle), ("objective", objective),
                          ("seed", seed), ("_pending", (assign_dev, members_dev, offsets))):
            object.__setattr__(self, name, val)
        self._dev()["assign"] = assign_dev

    def _host_lists(self):
        h = self.__dict__.get("_host_lists_")
        if h is None:
            assign_dev, members_dev, offsets = self._pending
            a_h, m_h = (x.copy() for x in _device.to_host_pinned_many(assign_dev, members_dev))
            a_h = a_h.astype(np.int64, copy=False)
            for x in (a_h, m_h):
                x.setflags(write=False)
            h = (a_h, tuple(m_h[offsets[c]:offsets[c + 1]] for c in range(offsets.shape[0] - 1)))
            object.__setattr__(self, "_host_lists_", h)
        return h

    @property
    def assignment(self) -> np.ndarray:
        return self._host_lists()[0]

    @property
    def members(self) -> tuple:
        return self._host_lists()[1]

    def num_assigned(self) -> int:
        return int(self._pending[0].shape[0])


def _half_angles(vectors: np.ndarray, center: np.ndarray) -> np.ndarray:
    cn = np.linalg.norm(center)
    if cn == 0.0:
        return np.full(vectors.shape[0], DEGENERATE_ANGLE)
    n = np.linalg.norm(vectors, axis=1)
    x = vectors / np.where(n > 0.0, n, 1.0)[:, None]
    y = center / cn
    a = 2.0 * np.arctan2(np.linalg.norm(x - y, axis=1), np.linalg.norm(x + y, axis=1))
    a[n == 0.0] = DEGENERATE_ANGLE
    return a


def angular_distance(a, b) -> float:
    """Angle in [0, pi] between two nonzero vectors, half-angle form
    2*atan2(|x-y|, |x+y|) on unit vectors (clustering.py:47-62).  A host
    scalar helper (two vectors), not part of the batched path."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if np.linalg.norm(a) == 0.0 or np.linalg.norm(b) == 0.0:
        raise ValueError("angular distance is undefined for zero-norm vectors")
    return float(_half_angles(a[None, :], b)[0])


def angles_to_center(vectors, center) -> np.ndarray:
    """Per-row angle to ``center``; degenerate rows (or center) get pi
    (clustering.py:65-78).  Host helper for inspection and tests."""
    return _half_angles(np.atleast_2d(np.asarray(vectors, dtype=np.float64)), np.asarray(center, dtype=np.float64))


def _as_matrix(x):
    return x if isinstance(x, FactorMatrix) else FactorMatrix(np.asarray(x, dtype=np.float64))


def compute_max_angles(users, centroids, assignment) -> np.ndarray:
    """theta_b per cluster: max member-to-centroid angle, 0 for empty clusters
    (clustering.py:81-93), computed on the GPU."""
    um, cm = _as_matrix(users), _as_matrix(centroids)
    a = _device.to_device(np.asarray(assignment, dtype=np.int64))
    return _device.to_host(_ops.max_angles(_device.f64(um), _device.f64(cm), a)).copy()


def _finish_seeds_on_degenerate(points_h, rows_h, start):
    """clustering.py:113-117: with a zero D^2 total, take the lowest-id point
    not already a seed (no RNG draw).  Once the total is zero it stays zero,
    so every remaining pass takes this branch."""
    n = points_h.shape[0]
    taken = {tuple(points_h[r]) for r in rows_h[:start]}
    for j in range(start, rows_h.shape[0]):
        pick = j % n
        for i in range(n):
            if tuple(points_h[i]) not in taken:
                pick = i
                break
        rows_h[j] = pick
        taken.add(tuple(points_h[pick]))
    return rows_h


def _repair_empty_host(points_h, centers_h, assign_h, d2_h):
    """clustering.py:125-138: an empty cluster takes the farthest point whose
    own cluster keeps at least one member.  Rare (only when a Lloyd step
    empties a cluster); runs on the host copies and is re-uploaded."""
    counts = np.bincount(assign_h, minlength=centers_h.shape[0])
    changed = False
    for c in np.flatnonzero(counts == 0):
        for cand in np.argsort(-d2_h, kind="stable"):
            cand = int(cand)
            if counts[assign_h[cand]] > 1:
                counts[assign_h[cand]] -= 1
                assign_h[cand] = c
                counts[c] = 1
                centers_h[c] = points_h[cand]
                d2_h[cand] = 0.0
                changed = True
                break
    return changed


def kmeans(users: FactorMatrix, num_clusters: int = DEFAULT_NUM_CLUSTERS, max_iters: int = DEFAULT_MAX_ITERS,
           seed: int = 0) -> Clustering:
    """Lloyd iterations with k-means++ seeding, stopping on a stable
    assignment (clustering.py:141-198).  Deterministic for a fixed seed; the
    RNG stream (and hence the seeds) is the reference's."""
    n = users.rows
    if not 1 <= num_clusters <= n:
        raise ValueError(f"num_clusters must be in [1, {n}], got {num_clusters}")
    if max_iters < 1:
        raise ValueError("max_iters must be >= 1")
    pts = _device.f64(users)
    dev = pts.device
    rng = np.random.default_rng(seed)
    first = int(rng.integers(0, n))
    unif = _device.to_device(rng.random(num_clusters - 1)) if num_clusters > 1 else None
    # (the draws are uploaded before f32_exact's flag read-back: the seeding
    # launch then follows that synchronisation at once)
    p32 = _device.f32_exact(users)  # exact float32 copy (half the bytes) or None
    rows, centers, deg = _ops.kmeans_seed(pts, num_clusters, first, unif, points32=p32)
    # the degenerate-seeding flag is read through a side stream while the first
    # assignment (queued at once, speculatively) runs: the host wait ends when
    # the seeding does, and the GPU does not idle while the loop is queued
    seeded = torch.cuda.Event()
    seeded.record()
    side = _device.side_stream(dev)
    deg_h = torch.empty(1, dtype=deg.dtype, pin_memory=True)
    with torch.cuda.stream(side):
        side.wait_event(seeded)
        deg_h.copy_(deg, non_blocking=True)
        deg_read = torch.cuda.Event()
        deg_read.record()
    deg.record_stream(side)

    def repair(assign_t, d2_t, counts_t):
        if not (_device.to_host(counts_t) == 0).any():
            return assign_t, False
        a_h = _device.to_host(assign_t).copy()
        c_h = _device.to_host(centers).copy()
        d_h = _device.to_host(d2_t).copy()
        _repair_empty_host(users.values, c_h, a_h, d_h)
        centers.copy_(torch.as_tensor(c_h, device=dev))
        return torch.as_tensor(a_h, device=dev), True

    tok = -next(_RUN_TOKENS)  # this run's assignments share the point side of the product (negative: not a query set's)
    assign, d2, _, obj = _ops.kmeans_assign(pts, centers, points32=p32, token=tok)
    deg_read.synchronize()
    deg_pass = int(deg_h.item())
    if deg_pass >= 0:  # fewer distinct points than seeds: finish on the host, redo the first assignment
        rows_h = _device.to_host(rows).copy()
        rows_h = _finish_seeds_on_degenerate(users.values, rows_h, deg_pass)
        centers = torch.as_tensor(users.values[rows_h], device=dev).contiguous()
        assign, d2, _, obj = _ops.kmeans_assign(pts, centers, points32=p32, token=tok)
    objs = [obj]  # read back once at the end (no per-iteration sync for the history)

    def lloyd_step(a_cur):
        counts, _, _ = _ops.kmeans_update(pts, a_cur, centers, points32=p32)
        new_assign, d_new, changed, ob = _ops.kmeans_assign(pts, centers, prev=a_cur, points32=p32, token=tok)
        flag = torch.stack([(counts == 0).any().to(torch.int64), changed.view(())])
        return counts, new_assign, d_new, flag, ob

    # Lloyd iterations in speculative batches with one host read per batch
    # ("a cluster went empty", "assignment changed" for every iteration of
    # the batch).  Iterations queued after convergence recompute the same
    # centres (means of the same assignment, deterministic) and the same
    # assignment, so the state is the converged one; only their objective
    # entries are dropped.  A batch in which a cluster went empty (rare) is
    # rolled back and replayed one iteration per read with the host repair
    # (clustering.py:125-138).
    it = 0
    done = False
    while it < max_iters and not done:
        batch = min(max_iters - it, _LLOYD_BATCH)
        snap = (assign.clone(), centers.clone(), d2) if batch > 1 else None
        steps, a_cur = [], assign
        for _ in range(batch):
            counts, new_assign, d_new, flag, ob = lloyd_step(a_cur)
            steps.append((a_cur, counts, new_assign, d_new, ob))
            a_cur = new_assign
            steps[-1] = steps[-1] + (flag,)
        flags = torch.stack([st[5] for st in steps]).tolist()
        used = next((i + 1 for i, (_, ch) in enumerate(flags) if ch == 0), batch)  # iterations that count
        if batch > 1 and any(e for e, _ in flags[:used]):
            # roll back and replay this batch one iteration per read, with the repair
            assign, d2 = snap[0], snap[2]
            centers.copy_(snap[1])
            for _ in range(batch):
                d2_before = d2
                counts, new_assign, d2, flag, ob = lloyd_step(assign)
                empty, n_changed = flag.tolist()
                if empty:
                    assign, _ = repair(assign, d2_before, counts)
                    new_assign, d2, changed, ob = _ops.kmeans_assign(pts, centers, prev=assign, points32=p32, token=tok)
                    n_changed = int(changed.item())
                objs.append(ob)
                it += 1
                if n_changed == 0:
                    done = True
                    break
                assign = new_assign
            continue
        if batch == 1 and flags[0][0]:  # a single iteration emptied a cluster: repair, redo the assignment
            a_prev, counts = steps[0][0], steps[0][1]
            assign, _ = repair(a_prev, d2, counts)
            new_assign, d2, changed, ob = _ops.kmeans_assign(pts, centers, prev=assign, points32=p32, token=tok)
            objs.append(ob)
            it += 1
            if int(changed.item()) == 0:
                done = True
            else:
                assign = new_assign
            continue
        for i in range(used):
            a_prev, _, new_assign, d_new, ob, _ = steps[i]
            objs.append(ob)
            d2 = d_new
            it += 1
            if flags[i][1] == 0:
                done = True
                assign = a_prev
                break
            assign = new_assign
    counts, members, offsets = _ops.kmeans_update(pts, assign, None, num_clusters)
    theta = _ops.max_angles(pts, centers, assign)
    cen_h, theta_h, off_h, objective = (a.copy() for a in _device.to_host_pinned_many(
        centers, theta, offsets, torch.cat(objs)))
    if (np.diff(off_h) == 0).any():  # rare: an empty cluster after the last iteration
        assign, fixed = repair(assign, d2, counts)
        counts, members, offsets = _ops.kmeans_update(pts, assign, None, num_clusters)
        theta = _ops.max_angles(pts, centers, assign)
        cen_h, theta_h, off_h = (a.copy() for a in _device.to_host_pinned_many(centers, theta, offsets))
    for a in (theta_h, objective):
        a.setflags(write=False)
    cen_fm = FactorMatrix(cen_h)
    _device._cache(cen_fm)["f64"] = centers  # resident already: build_index reads it without an upload
    out = _DeviceClustering(cen_fm, theta_h, objective, seed, assign.contiguous(), members, off_h)
    out._dev()["theta"] = theta
    return out
