"""GPU tests of the k-means kernels against numpy restatements of
clustering.py: the tensor-core assignment (certified band + float64
rescoring) and its SIMT fallback, the counting-sort grouping and in-order
centroid sums of the update step (bit-identical to numpy's mean), and the
persistent k-means++ seeding (triangle skip, factor-order distances) against
the oracle's draw-for-draw seeding, including the degenerate (duplicate
points) branch."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_01449_b200 as pkg
    from paper_1706_01449_b200 import _ops
    return pkg, _ops, torch


def _dev(torch, a):
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda")


def _np_assign(points, centers):
    """clustering.py:96-101 in float64: (p2 + c2) - 2 p.c, clipped, first argmin."""
    p2 = (points * points).sum(axis=1)
    c2 = (centers * centers).sum(axis=1)
    d2 = np.maximum(p2[:, None] + c2[None, :] - 2.0 * (points @ centers.T), 0.0)
    return d2.argmin(axis=1), d2


@pytest.mark.parametrize("n,f,c", [(5000, 50, 256), (3000, 7, 3), (2000, 255, 40), (2000, 256, 40),
                                   (700, 1, 9), (4100, 64, 1000)])
def test_assign_matches_float64_argmin(env, n, f, c):
    pkg, _ops, torch = env
    rng = np.random.default_rng(n + f + c)
    centers = rng.normal(size=(c, f))
    comp = rng.integers(0, c, n)
    points = centers[comp] + 0.3 * rng.normal(size=(n, f))
    centers[1 % c] = centers[0]  # duplicate centres: equal distances, first index must win
    a, d2, _, obj = _ops.kmeans_assign(_dev(torch, points), _dev(torch, centers))
    want, d2_all = _np_assign(points, centers)
    got = a.cpu().numpy()
    best = d2_all[np.arange(n), want]
    # the pick must be a float64 minimiser; exact index equality away from ulp-level ties
    np.testing.assert_allclose(d2_all[np.arange(n), got], best, rtol=1e-12, atol=1e-12)
    clear = np.sort(d2_all, axis=1)
    clear = (clear[:, 1] - clear[:, 0]) > 1e-9 * (1.0 + clear[:, 0]) if c > 1 else np.ones(n, bool)
    assert np.array_equal(got[clear], want[clear])
    np.testing.assert_allclose(d2.cpu().numpy(), best, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(float(obj.item()), best.sum(), rtol=1e-12)


def test_assign_float32_copy_path(env):
    """The exact float32 copy (BASELINE inputs are float32) gives the same answer."""
    pkg, _ops, torch = env
    rng = np.random.default_rng(5)
    points = rng.normal(size=(6000, 50)).astype(np.float32).astype(np.float64)
    centers = points[rng.choice(6000, 100, replace=False)]
    p = _dev(torch, points)
    p32, exact = _ops.to_f32(p)
    assert exact
    a64, d64, _, _ = _ops.kmeans_assign(p, _dev(torch, centers))
    a32, d32, _, _ = _ops.kmeans_assign(p, _dev(torch, centers), points32=p32)
    assert torch.equal(a64, a32)
    assert torch.equal(d64, d32)


@pytest.mark.parametrize("n,c", [(10000, 7), (20000, 300), (20000, 9000)])
def test_update_groups_stably_and_means(env, n, c):
    """Counting-sort grouping (and the sort fallback for c > 8192): members in
    (cluster, id) order, counts/offsets, centroid means; empty clusters keep
    their centroid (clustering.py:169-172)."""
    pkg, _ops, torch = env
    rng = np.random.default_rng(n + c)
    f = 13
    points = rng.normal(size=(n, f))
    assign = rng.integers(0, c, n)
    assign[assign == 1] = 0  # cluster 1 empty
    centers = rng.normal(size=(c, f))
    cen_t = _dev(torch, centers.copy())
    counts, members, offsets = _ops.kmeans_update(_dev(torch, points), _dev(torch, assign.astype(np.int64)), cen_t)
    order = np.argsort(assign, kind="stable")
    np.testing.assert_array_equal(members.cpu().numpy(), order)
    want_counts = np.bincount(assign, minlength=c)
    np.testing.assert_array_equal(counts.cpu().numpy(), want_counts)
    np.testing.assert_array_equal(offsets.cpu().numpy(), np.concatenate([[0], np.cumsum(want_counts)]))
    got = cen_t.cpu().numpy()
    for j in range(c):
        want = points[assign == j].mean(axis=0) if want_counts[j] else centers[j]
        np.testing.assert_array_equal(got[j], want)  # sequential row sums, then one divide


@pytest.mark.parametrize("n,f,k,dtype", [(20000, 50, 64, np.float32), (5000, 17, 200, np.float64),
                                         (3000, 128, 30, np.float32), (40000, 8, 16, np.float64)])
def test_seeding_matches_oracle_draws(env, n, f, k, dtype):
    """Persistent seeding picks the oracle's rows (same RNG draws, same D^2)."""
    pkg, _ops, torch = env
    import simdex_oracle as O
    rng = np.random.default_rng(n + k)
    centers = rng.normal(size=(max(k // 2, 1), f))
    users = (centers[rng.integers(0, centers.shape[0], n)] + 0.2 * rng.normal(size=(n, f))).astype(dtype)
    users = users.astype(np.float64)
    seed = 7
    r1 = np.random.default_rng(seed)
    want = O.plusplus_seeds(users, k, r1)
    r2 = np.random.default_rng(seed)
    first = int(r2.integers(0, n))
    unif = _dev(torch, r2.random(k - 1))
    p = _dev(torch, users)
    p32, exact = _ops.to_f32(p)
    rows, cen, deg = _ops.kmeans_seed(p, k, first, unif, points32=p32 if exact else None)
    assert int(deg.item()) < 0
    np.testing.assert_array_equal(cen.cpu().numpy(), want)


def test_seeding_degenerate_branch(env):
    """Fewer distinct points than seeds (clustering.py:113-117 and the empty
    cluster repair): the clustering still equals the oracle's."""
    pkg, _ops, torch = env
    rng = np.random.default_rng(3)
    base = rng.normal(size=(4, 6))
    users = base[rng.integers(0, 4, 500)]
    cl = pkg.kmeans(pkg.FactorMatrix(users), 6, max_iters=5, seed=2)
    import simdex_oracle as O
    ref = O.kmeans(users, 6, max_iters=5, seed=2)
    np.testing.assert_array_equal(cl.assignment, ref["assignment"])


@pytest.mark.parametrize("n,f,c,iters,seed", [(3000, 8, 20, 7, 1), (2000, 50, 64, 3, 4), (800, 3, 40, 100, 9),
                                             (500, 6, 6, 5, 2)])
def test_lloyd_batches_equal_sequential(env, n, f, c, iters, seed):
    """Lloyd iterations queued in speculative batches (one host read per
    batch) give exactly the sequential loop's clustering: assignment,
    centroids, objective history (iterations after convergence dropped) and
    theta_b; also against the oracle's restatement of clustering.py."""
    pkg, _ops, torch = env
    from paper_1706_01449_b200 import clustering
    rng = np.random.default_rng(seed)
    if seed == 2:  # duplicates: the degenerate seeding branch and the final repair
        users = rng.normal(size=(4, f))[rng.integers(0, 4, n)]
    else:
        users = rng.normal(size=(n, f)) * rng.lognormal(0.0, 1.0, size=(n, 1))
    m = pkg.FactorMatrix(users)
    old = clustering._LLOYD_BATCH
    try:
        clustering._LLOYD_BATCH = 1
        a = pkg.kmeans(m, c, max_iters=iters, seed=seed)
        clustering._LLOYD_BATCH = 3
        b = pkg.kmeans(pkg.FactorMatrix(users), c, max_iters=iters, seed=seed)
    finally:
        clustering._LLOYD_BATCH = old
    np.testing.assert_array_equal(a.assignment, b.assignment)
    np.testing.assert_array_equal(a.centroids.values, b.centroids.values)
    np.testing.assert_array_equal(a.objective, b.objective)
    np.testing.assert_array_equal(a.max_angle, b.max_angle)
    import simdex_oracle as O
    ref = O.kmeans(users, c, max_iters=iters, seed=seed)
    np.testing.assert_array_equal(b.assignment, ref["assignment"])
    assert b.objective.shape == ref["objective"].shape


def test_assign_reuses_point_side_under_a_token(env):
    """Consecutive assignments over the same points under one context token
    (the Lloyd loop) skip the point side of the product; the results are those
    of untagged calls, for changed centres too, and another call on the
    context in between invalidates the held setup."""
    pkg, _ops, torch = env
    rng = np.random.default_rng(5)
    n, f, c = 40000, 24, 64
    centers = rng.normal(size=(c, f))
    points = (centers[rng.integers(0, c, n)] + 0.4 * rng.normal(size=(n, f))).astype(np.float32).astype(np.float64)
    pts = _dev(torch, points)
    p32 = pts.to(torch.float32)
    tok = -987654
    for it in range(4):
        cen = _dev(torch, centers + 0.05 * it * rng.normal(size=(c, f)))
        a0, d0, _, o0 = _ops.kmeans_assign(pts, cen, points32=p32)
        a1, d1, _, o1 = _ops.kmeans_assign(pts, cen, points32=p32, token=tok)
        assert torch.equal(a0, a1) and torch.equal(d0, d1) and torch.equal(o0, o1)
        if it == 2:  # a different problem on the same context: the held point side must not be reused after it
            other = _dev(torch, rng.normal(size=(n, f)))
            _ops.kmeans_assign(other, cen)
    want, _ = _np_assign(points, cen.cpu().numpy())
    assert np.array_equal(a1.cpu().numpy(), want)
