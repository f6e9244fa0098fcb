"""GPU tests of the tensor-core path: raw tcgen05 accumulators against a
float32 torch reference, the certified top-K against the exact float64 scan
over many shapes, work sharing against the plain walk, and the BASELINE cfg2
workload at full size against the reference's golden answers."""

import numpy as np
import pytest

from conftest import assert_same_topk, load_golden, near_tie_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1706_01449_b200 as pkg
    return pkg


def _model(sx, users, items):
    return sx.ModelPair(sx.FactorMatrix(users), sx.FactorMatrix(items))


@pytest.mark.parametrize("nu,ni,f", [(300, 500, 50), (256, 128, 64), (1000, 77, 5), (130, 1300, 100),
                                     (513, 260, 128), (40, 33, 1), (260, 300, 200)])
def test_tcgen05_accumulators_match_float_reference(sx, nu, ni, f):
    """The raw TMEM accumulators equal fp32 products of the fp16 operands."""
    import torch
    from paper_1706_01449_b200 import _device, _ops
    rng = np.random.default_rng(nu * 7 + f)
    m = _model(sx, rng.normal(size=(nu, f)), rng.normal(size=(ni, f)) * rng.lognormal(0, 1, (ni, 1)))
    pu, pi = _device.packed(m.users), _device.packed(m.items)
    got = _ops.gemm_debug(pu, pi, f)
    a = _f16_to_f32(pu.op[:nu, :f])
    b = _f16_to_f32(pi.op[:ni, :f])
    want = (a.double() @ b.double().T)
    scale = (a.double().abs() @ b.double().abs().T)
    err = (got.double() - want).abs()
    assert bool((err <= scale * (f + 2) * 2.0 ** -22 + 1e-30).all()), float((err / scale.clamp_min(1e-30)).max())


def _f16_to_f32(t16):
    import torch
    return t16.view(torch.float16).float()


@pytest.mark.parametrize("nu,ni,f,k", [(700, 2000, 50, 10), (300, 129, 8, 1), (257, 4000, 32, 100), (100, 50, 3, 5),
                                       (260, 1000, 128, 256), (512, 700, 100, 50), (64, 300, 1, 7),
                                       (300, 5000, 16, 200)])
def test_certified_topk_equals_exact(sx, nu, ni, f, k):
    rng = np.random.default_rng(nu + ni + f + k)
    users = rng.normal(size=(nu, f)) * rng.uniform(0.1, 3.0, (nu, 1))
    items = rng.normal(size=(ni, f)) * rng.lognormal(0, 0.7, (ni, 1))
    m = _model(sx, users, items)
    fast = sx.topk_matmul(m, k)
    ref = sx.topk_naive(m, k)
    assert_same_topk(fast.item_ids, fast.scores, ref.item_ids, ref.scores, ctx=f"{nu}x{ni}x{f} k={k}")


def test_certified_topk_with_exact_ties(sx):
    """Duplicated item rows and integer-valued data: exact score ties resolved by id."""
    rng = np.random.default_rng(5)
    base = rng.integers(-3, 4, size=(300, 6)).astype(float)
    items = np.vstack([base, base[::3]])
    users = rng.integers(-2, 3, size=(400, 6)).astype(float)
    m = _model(sx, users, items)
    for k in (1, 7, 40):
        fast = sx.topk_matmul(m, k)
        ref = sx.topk_naive(m, k)
        assert_same_topk(fast.item_ids, fast.scores, ref.item_ids, ref.scores, ctx=f"ties k={k}")


def test_heap_ops_monotone_in_k(sx):
    m = sx.generate_synthetic(sx.SyntheticSpec(600, 2500, 6, seed=6))
    totals = []
    for k in (1, 5, 10, 50):
        cnt = {}
        sx.topk_matmul(m, k, counters=cnt)
        totals.append(int(cnt["heap_ops"].sum()))
    assert totals == sorted(totals) and totals[0] < totals[-1]


@pytest.mark.parametrize("block", [1, 64, 300, 4096])
def test_work_sharing_equals_walk(sx, block):
    m = sx.generate_synthetic(sx.SyntheticSpec(3000, 6000, 24, archetype_count=12, angular_spread=0.25,
                                               norm_low=0.5, norm_high=2.5, seed=17))
    cl = sx.kmeans(m.users, 12, seed=2)
    idx = sx.build_index(m, cl, block)
    for k in (1, 10, 64):
        on = sx.query_batch(idx, m, None, k, work_sharing=True)
        off = sx.query_batch(idx, m, None, k, work_sharing=False)
        assert_same_topk(on.item_ids, on.scores, off.item_ids, off.scores, ctx=f"B={block} k={k}")
        np.testing.assert_array_equal(on.visited, np.maximum(min(block, m.num_items), off.visited))
        sub = [5, 2999, 17, 5, 1200]
        part = sx.query_batch(idx, m, sub, k, work_sharing=True)
        np.testing.assert_array_equal(part.item_ids, on.item_ids[sub])
        np.testing.assert_array_equal(part.visited, on.visited[sub])


def test_cfg2_full_size_against_reference(sx):
    """BASELINE configs[1] at full size (480,189 x 17,770, f=50): the GPU
    k-means reproduces the reference clustering, and the work-sharing serve
    path returns the reference's ids, scores and visited counts on a 2,000
    user sample for K in {1, 5, 10, 50} (every BASELINE depth)."""
    from paper_1706_01449_b200 import workloads as W
    g = load_golden("cfg2_index")
    w = W.cfg2()
    m = _model(sx, w.users, w.items)
    cl = sx.kmeans(m.users, 256, max_iters=3, seed=1)
    same = float((cl.assignment == g["assignment"].astype(np.int64)).mean())
    assert same == 1.0, f"assignment agreement {same}"
    np.testing.assert_array_equal(cl.centroids.values, g["centroids"])  # in-order sums: bit-identical
    np.testing.assert_allclose(cl.max_angle, g["max_angle"], rtol=1e-10)
    np.testing.assert_allclose(cl.objective, g["objective"], rtol=1e-10)
    idx = sx.build_index(m, cl, 4096)
    np.testing.assert_array_equal(idx.item_ids[:, :64], g["ids_head"].astype(np.int64))
    np.testing.assert_allclose(idx.bounds[:, :64], g["bounds_head"], rtol=1e-12)
    sample = g["sample"]
    for k in (1, 5, 10, 50):
        res = sx.query_batch(idx, m, sample, k, work_sharing=True)
        want_ids = g[f"ws_k{k}_ids"].astype(np.int64)
        assert_same_topk(res.item_ids, res.scores, want_ids, g[f"ws_k{k}_scores"], ctx=f"cfg2 k={k}")
        np.testing.assert_array_equal(res.visited, g[f"ws_k{k}_visited"])
        nows = sx.query_batch(idx, m, sample[:500], k, work_sharing=False)
        np.testing.assert_array_equal(nows.visited, g[f"nows_k{k}_visited"])
    # the same answers with the prefix pass's ceiling exit forced on (it is
    # normally enabled only when the walk estimate is short against B)
    from paper_1706_01449_b200 import index as I
    for k in (1, 5, 10, 50):
        I.note_walk_estimate(idx, k, 0.0)
        res = sx.query_batch(idx, m, sample, k, work_sharing=True)
        assert_same_topk(res.item_ids, res.scores, g[f"ws_k{k}_ids"].astype(np.int64), g[f"ws_k{k}_scores"],
                         ctx=f"cfg2 k={k} prefix exit")
        np.testing.assert_array_equal(res.visited, g[f"ws_k{k}_visited"])
        idx._dev.pop(("walk_estimate", k))
        est = sx.estimate_walk_length(idx, m, 0.001, k, seed=1)
        np.testing.assert_allclose([est.mean_visited, est.ci_low, est.ci_high, est.sample_size], g[f"est_k{k}"],
                                   rtol=1e-12)


@pytest.mark.parametrize("n", [1, 2, 7, 2047, 2048, 2049, 4097, 17770, 100003])
def test_norm_order_sort_matches_lexsort(n):
    """simdex_norm_order (the merge sort every list build uses): (value desc,
    id asc) with many exact ties and signed zeros, against numpy's lexsort."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1706_01449_b200 import _lib
    from paper_1706_01449_b200._lib import stream_ptr
    rng = np.random.default_rng(n)
    v = rng.integers(0, max(2, n // 5), n).astype(np.float64) * 0.25
    v[rng.random(n) < 0.1] = -0.0
    v[rng.random(n) < 0.1] = 0.0
    d = torch.as_tensor(v, device="cuda")
    perm = torch.empty(n, dtype=torch.int32, device="cuda")
    _lib.call("simdex_norm_order", d.data_ptr(), n, perm.data_ptr(), stream_ptr())
    want = np.lexsort((np.arange(n), -v))
    np.testing.assert_array_equal(perm.cpu().numpy(), want)


@pytest.mark.parametrize("ni,c,f", [(5000, 7, 13), (4096, 3, 50), (9000, 20, 8)])
def test_build_index_lists_match_oracle(ni, c, f):
    """Eq. 2 ceilings and the (ceiling desc, id asc) lists at sizes that take
    the merge passes, against the oracle's build_index (its numpy norms sum
    pairwise, so ceilings agree to ~1e-12; the order is checked exactly)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import simdex_oracle as O
    from paper_1706_01449_b200 import _ops
    rng = np.random.default_rng(ni + c)
    items = rng.normal(size=(ni, f)) * rng.lognormal(0, 0.5, ni)[:, None]
    items[3] = 0.0  # zero item: angle pi/2, ceiling 0
    items[ni // 2] = items[ni // 3]  # duplicate rows: equal ceilings, id order
    centers = rng.normal(size=(c, f))
    theta = rng.uniform(0.0, 1.2, c)
    norms, ids, bounds = _ops.build_index(torch.as_tensor(items, device="cuda"), torch.as_tensor(centers, device="cuda"),
                                          torch.as_tensor(theta, device="cuda"))
    want_ids, want_b, want_norms = O.build_index(items, centers, theta)
    got_ids, got_b = ids.cpu().numpy().astype(np.int64), bounds.cpu().numpy()
    np.testing.assert_allclose(norms.cpu().numpy(), want_norms, rtol=1e-14)
    for r in range(c):
        # a permutation in (ceiling desc, id asc) order of its own ceilings ...
        assert np.array_equal(np.sort(got_ids[r]), np.arange(ni))
        order = np.lexsort((got_ids[r], -got_b[r]))
        np.testing.assert_array_equal(order, np.arange(ni))
        # ... whose ceilings are the oracle's, item by item
        by_item = np.empty(ni)
        by_item[got_ids[r]] = got_b[r]
        want_item = np.empty(ni)
        want_item[want_ids[r]] = want_b[r]
        np.testing.assert_allclose(by_item, want_item, rtol=1e-12, atol=1e-13)  # cos near 0: absolute
