"""Tensor-level wrappers of the C-ABI (device in, device out).

Each function allocates its outputs with torch (the caching allocator is the
plumbing), validates shapes, and enqueues the library call on the current
stream.  Nothing here computes on the host.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import call, ptr, stream_ptr

F64 = torch.float64
I64 = torch.int64
I32 = torch.int32


def _dev():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _c(t, dtype):
    assert t.dtype == dtype and t.is_cuda and t.is_contiguous(), (t.dtype, t.device, t.is_contiguous())
    return t


@dataclass
class Packed:
    """fp16 tensor-core operand of a factor matrix (see simdex_pack_f16)."""

    op: torch.Tensor        # fp16 bits in int16 storage [rows_pad, kp]
    norms: torch.Tensor     # float64 [rows] norms of the unscaled rows
    scale_exp: int
    kp: int
    rows: int
    perm: torch.Tensor | None = None   # operand row -> item id (norm-sorted operand), else None
    rows_pad: int = 0                  # rows of the fp16 operand
    norm_exit: bool = False            # norm-sorted and skewed enough for the brute-force early exit
    row_exp: torch.Tensor | None = None  # int32 [rows]: per-row scale exponents (pack_rows), else None


ROW_PAD = 256


def norm_sorted(p: Packed) -> Packed:
    """The item operand re-laid out by (norm desc, id asc) (simdex_norm_order):
    the brute-force pass then meets high-norm items first, its thresholds rise
    early and low-norm tiles fail the norm bound."""
    perm = torch.empty(p.rows, dtype=I32, device=p.op.device)
    call("simdex_norm_order", ptr(p.norms), p.rows, ptr(perm), stream_ptr())
    rows_pad = ROW_PAD * ((p.rows + ROW_PAD - 1) // ROW_PAD)
    out = torch.empty((1, rows_pad, p.kp), dtype=torch.int16, device=p.op.device)
    onorm = torch.empty((1, rows_pad), dtype=F64, device=p.op.device)
    call("simdex_build_prefix", ptr(p.op), ptr(p.norms), p.rows, p.kp, ptr(perm), 1, p.rows, rows_pad, ptr(out),
         ptr(onorm), stream_ptr())
    # the exit's extra control flow costs ~14 % where nothing can be skipped
    # (i.i.d. norms); decided once per operand from the largest and median norm
    top, mid = (float(v) for v in onorm.view(-1)[torch.tensor([0, p.rows // 2], device=onorm.device)].tolist())
    skewed = p.rows >= 256 and mid < 0.6 * top
    return Packed(out.view(rows_pad, p.kp), onorm.view(rows_pad), p.scale_exp, p.kp, p.rows, perm, rows_pad, skewed)


def pack(x: torch.Tensor, max_abs: float) -> Packed:
    """fp16 copy scaled by 2^e so that the largest |entry| lies in [1, 2)."""
    rows, f = x.shape
    e = 0 if max_abs == 0.0 else -int(math.floor(math.log2(max_abs)))
    kp = 64 * ((f + 63) // 64)
    rows_pad = ROW_PAD * ((rows + ROW_PAD - 1) // ROW_PAD)
    out = torch.empty((rows_pad, kp), dtype=torch.int16, device=x.device)
    norms = torch.empty(rows, dtype=F64, device=x.device)
    call("simdex_pack_f16", ptr(_c(x, F64)), rows, f, e, rows_pad, kp, ptr(out), ptr(norms), stream_ptr())
    return Packed(out, norms, e, kp, rows)


def pack_rows(x: torch.Tensor) -> Packed:
    """fp16 copy with one exact power-of-two scale per row (max |entry| of
    every row in [1, 2)): the user operand (simdex_pack_f16_rows)."""
    rows, f = x.shape
    kp = 64 * ((f + 63) // 64)
    rows_pad = ROW_PAD * ((rows + ROW_PAD - 1) // ROW_PAD)
    out = torch.empty((rows_pad, kp), dtype=torch.int16, device=x.device)
    norms = torch.empty(rows, dtype=F64, device=x.device)
    row_exp = torch.empty(rows, dtype=I32, device=x.device)
    call("simdex_pack_f16_rows", ptr(_c(x, F64)), rows, f, rows_pad, kp, ptr(out), ptr(norms), ptr(row_exp),
         stream_ptr())
    return Packed(out, norms, 0, kp, rows, row_exp=row_exp)


def topk_exact(users, items, k, rows=None):
    nu, f = users.shape
    ni = items.shape[0]
    k_eff = min(k, ni)
    n_rows = nu if rows is None else rows.shape[0]
    ids = torch.empty((n_rows, k_eff), dtype=I32, device=users.device)
    sc = torch.empty((n_rows, k_eff), dtype=F64, device=users.device)
    call("simdex_topk_exact", ptr(_c(users, F64)), nu, ptr(_c(items, F64)), ni, f,
         ptr(None if rows is None else _c(rows, I64)), n_rows, k, ptr(ids), ptr(sc), stream_ptr())
    return ids, sc


def topk_matmul(users, pu: Packed, items, pi: Packed, k, heap_ops=False, items32=None, users32=None, ctx=None):
    nu, f = users.shape
    ni = items.shape[0]
    k_eff = min(k, ni)
    ids = torch.empty((nu, k_eff), dtype=I32, device=users.device)
    sc = torch.empty((nu, k_eff), dtype=F64, device=users.device)
    hops = torch.zeros(nu, dtype=I64, device=users.device) if heap_ops else None
    call("simdex_topk_matmul_ctx", ctx, ptr(_c(users, F64)), ptr(users32), ptr(pu.op), ptr(pu.norms), nu,
         ptr(_c(items, F64)), ptr(items32), ptr(pi.op), ptr(pi.norms), ptr(pi.perm), pi.rows_pad, ni, f, pu.kp,
         pu.scale_exp, ptr(pu.row_exp), pi.scale_exp, k, ptr(ids), ptr(sc), ptr(hops),
         MM_NORM_EXIT if pi.norm_exit else 0, stream_ptr())
    return ids, sc, hops


def max_abs(x) -> float:
    out = torch.empty(1, dtype=F64, device=x.device)
    call("simdex_max_abs", ptr(_c(x, F64)), x.numel(), ptr(out), stream_ptr())
    return float(out.item())


def to_f32(x):
    """(float32 copy, exact?) of a float64 tensor."""
    out = torch.empty(x.shape, dtype=torch.float32, device=x.device)
    flag = torch.empty(1, dtype=I32, device=x.device)
    call("simdex_to_f32", ptr(_c(x, F64)), x.numel(), ptr(out), ptr(flag), stream_ptr())
    return out, int(flag.item()) == 0


def kmeans_seed(points, k, first, uniforms, points32=None):
    n, f = points.shape
    rows = torch.empty(k, dtype=I64, device=points.device)
    centers = torch.zeros((k, f), dtype=F64, device=points.device)  # (defined rows even when the seeding stops early)
    deg = torch.empty(1, dtype=I32, device=points.device)
    call("simdex_kmeans_seed", ptr(_c(points, F64)), ptr(points32), n, f, k, int(first),
         ptr(None if uniforms is None else _c(uniforms, F64)), ptr(rows), ptr(centers), ptr(deg), stream_ptr())
    return rows, centers, deg


def kmeans_assign(points, centers, prev=None, points32=None, token=0):
    """``token`` != 0 (unique to one run over fixed points, e.g. a Lloyd loop):
    tags the thread's default context so that consecutive assignments reuse
    the point side of the product (simdex_ctx_set_query_token)."""
    n, f = points.shape
    c = centers.shape[0]
    assign = torch.empty(n, dtype=I64, device=points.device)
    d2 = torch.empty(n, dtype=F64, device=points.device)
    changed = torch.empty(1, dtype=I64, device=points.device)
    obj = torch.empty(1, dtype=F64, device=points.device)
    if token:
        call("simdex_ctx_set_query_token", None, C.c_int64(token))
    call("simdex_kmeans_assign", ptr(_c(points, F64)), ptr(points32), n, f, ptr(_c(centers, F64)), c,
         ptr(None if prev is None else _c(prev, I64)), ptr(assign), ptr(d2), ptr(changed), ptr(obj), stream_ptr())
    return assign, d2, changed, obj


def kmeans_update(points, assign, centers, c=None, points32=None):
    """Group users by cluster; with ``centers`` also recompute the means in place."""
    n, f = points.shape
    c = centers.shape[0] if centers is not None else c
    counts = torch.empty(c, dtype=I64, device=points.device)
    members = torch.empty(n, dtype=I64, device=points.device)
    offsets = torch.empty(c + 1, dtype=I64, device=points.device)
    call("simdex_kmeans_update", ptr(_c(points, F64)), ptr(points32), n, f, ptr(_c(assign, I64)), c,
         ptr(None if centers is None else _c(centers, F64)), ptr(counts), ptr(members), ptr(offsets), stream_ptr())
    return counts, members, offsets


def max_angles(users, centers, assign):
    n, f = users.shape
    c = centers.shape[0]
    theta = torch.empty(c, dtype=F64, device=users.device)
    call("simdex_max_angles", ptr(_c(users, F64)), n, f, ptr(_c(centers, F64)), c, ptr(_c(assign, I64)),
         ptr(theta), stream_ptr())
    return theta


def build_index(items, centers, theta, with_pos=False):
    """(item norms, list ids [c, n], ceilings [c, n][, inverse positions [c, n]])."""
    ni, f = items.shape
    c = centers.shape[0]
    norms = torch.empty(ni, dtype=F64, device=items.device)
    ids = torch.empty((c, ni), dtype=I32, device=items.device)
    bounds = torch.empty((c, ni), dtype=F64, device=items.device)
    pos = torch.empty((c, ni), dtype=I32, device=items.device) if with_pos else None
    call("simdex_build_index", ptr(_c(items, F64)), ni, f, ptr(_c(centers, F64)), ptr(_c(theta, F64)), c,
         ptr(norms), ptr(ids), ptr(bounds), ptr(pos), stream_ptr())
    return (norms, ids, bounds, pos) if with_pos else (norms, ids, bounds)


def list_positions(list_ids):
    c, ni = list_ids.shape
    pos = torch.empty((c, ni), dtype=I32, device=list_ids.device)
    call("simdex_list_positions", ptr(_c(list_ids, I32)), c, ni, ptr(pos), stream_ptr())
    return pos


def walk(users, unorm, items, list_ids, bounds, q_user, q_cluster, k, start=0, warm=None, no_prune=False,
         users32=None, items32=None):
    nq = q_user.shape[0]
    ni, f = items.shape
    k_eff = min(k, ni)
    ids = torch.empty((nq, k_eff), dtype=I32, device=users.device)
    sc = torch.empty((nq, k_eff), dtype=F64, device=users.device)
    vis = torch.empty(nq, dtype=I64, device=users.device)
    wi = ws = wc = None
    if warm is not None:
        wi, ws, wc = (_c(warm[0], I32), _c(warm[1], F64), _c(warm[2], I32))
    call("simdex_walk32", ptr(_c(users, F64)), ptr(_c(unorm, F64)), ptr(_c(items, F64)), ptr(users32), ptr(items32),
         f, ni, ptr(_c(list_ids, I32)), ptr(_c(bounds, F64)), ptr(_c(q_user, I64)), ptr(_c(q_cluster, I32)), nq, k,
         int(start), ptr(wi), ptr(ws), ptr(wc), int(bool(no_prune)), ptr(ids), ptr(sc), ptr(vis), stream_ptr())
    return ids, sc, vis


def build_prefix(pi: Packed, list_ids, block):
    """Per-cluster prefix operands: (fp16 [c, b_pad, kp], float64 norms [c, b_pad], b_pad)."""
    c, ni = list_ids.shape
    bp = min(block, ni)
    b_pad = 128 * ((bp + 127) // 128)
    out = torch.empty((c, b_pad, pi.kp), dtype=torch.int16, device=list_ids.device)
    onorm = torch.empty((c, b_pad), dtype=F64, device=list_ids.device)
    call("simdex_build_prefix", ptr(pi.op), ptr(pi.norms), ni, pi.kp, ptr(_c(list_ids, I32)), c, int(block),
         b_pad, ptr(out), ptr(onorm), stream_ptr())
    return out, onorm, b_pad


def build_prefix_ordered(pi: Packed, items, centers, list_ids, list_pos, bounds, block):
    """Per-cluster prefix operands in the centroid's score order:
    (fp16 [c, b_pad, kp], float64 norms [c, b_pad], b_pad, item ids int32
    [c, b_pad], per-tile ceiling bounds float64 [c, b_pad/128])."""
    c, ni = list_ids.shape
    f = items.shape[1]
    bp = min(block, ni)
    b_pad = 128 * ((bp + 127) // 128)
    dev = list_ids.device
    out = torch.empty((c, b_pad, pi.kp), dtype=torch.int16, device=dev)
    onorm = torch.empty((c, b_pad), dtype=F64, device=dev)
    ids = torch.empty((c, b_pad), dtype=I32, device=dev)
    tile_ceil = torch.empty((c, b_pad // 128), dtype=F64, device=dev)
    call("simdex_build_prefix_ordered", ptr(pi.op), ptr(pi.norms), ni, pi.kp, ptr(_c(items, F64)), f,
         ptr(_c(centers, F64)), ptr(_c(list_ids, I32)), ptr(_c(list_pos, I32)), ptr(_c(bounds, F64)), c, int(block),
         b_pad, ptr(out), ptr(onorm), ptr(ids), ptr(tile_ceil), stream_ptr())
    return out, onorm, b_pad, ids, tile_ceil


def build_prefix_hybrid(pi: Packed, items, centers, list_ids, list_pos, bounds, block, head):
    """build_prefix_ordered with the best ``head`` items (centroid score)
    first and the rest of the prefix in list order (simdex_build_prefix_hybrid)."""
    c, ni = list_ids.shape
    f = items.shape[1]
    bp = min(block, ni)
    b_pad = 128 * ((bp + 127) // 128)
    dev = list_ids.device
    out = torch.empty((c, b_pad, pi.kp), dtype=torch.int16, device=dev)
    onorm = torch.empty((c, b_pad), dtype=F64, device=dev)
    ids = torch.empty((c, b_pad), dtype=I32, device=dev)
    tile_ceil = torch.empty((c, b_pad // 128), dtype=F64, device=dev)
    call("simdex_build_prefix_hybrid", ptr(pi.op), ptr(pi.norms), ni, pi.kp, ptr(_c(items, F64)), f,
         ptr(_c(centers, F64)), ptr(_c(list_ids, I32)), ptr(_c(list_pos, I32)), ptr(_c(bounds, F64)), c, int(block),
         b_pad, int(head), ptr(out), ptr(onorm), ptr(ids), ptr(tile_ceil), stream_ptr())
    return out, onorm, b_pad, ids, tile_ceil


def group_queries(q_user, assign, c):
    """(grouped user rows, original positions, cluster offsets [c+1])."""
    nq = q_user.shape[0]
    gq = torch.empty(nq, dtype=I64, device=q_user.device)
    perm = torch.empty(nq, dtype=I64, device=q_user.device)
    off = torch.empty(c + 1, dtype=I64, device=q_user.device)
    call("simdex_group_queries", ptr(_c(q_user, I64)), nq, ptr(_c(assign, I64)), c, ptr(gq), ptr(perm), ptr(off),
         stream_ptr())
    return gq, perm, off


WS_PREFIX_EXIT = 1  # SIMDEX_WS_PREFIX_EXIT
MM_NORM_EXIT = 2    # SIMDEX_MM_NORM_EXIT


def query_ws(users, pu: Packed, items, pi: Packed, list_ids, list_pos, bounds, block, prefix, grouped, k,
             items32=None, users32=None, options=0, ctx=None):
    """Work-sharing batch query; ``grouped`` = group_queries(...) output.
    Returns (ids, scores, visited) in the original query order.  ``options``:
    WS_PREFIX_EXIT ends prefix units early on the list ceilings."""
    nu, f = users.shape
    ni = items.shape[0]
    c = list_ids.shape[0]
    gq, perm, off = grouped
    nq = gq.shape[0]
    k_eff = min(k, ni)
    ids = torch.empty((nq, k_eff), dtype=I32, device=users.device)
    sc = torch.empty((nq, k_eff), dtype=F64, device=users.device)
    vis = torch.empty(nq, dtype=I64, device=users.device)
    pb, pn, b_pad = prefix[:3]
    p_ids, p_ceil = prefix[3:5] if len(prefix) >= 5 else (None, None)
    call("simdex_query_ws_ctx", ctx, ptr(_c(users, F64)), ptr(users32), ptr(pu.op), ptr(pu.norms), nu, ptr(_c(items, F64)),
         ptr(items32),
         ptr(pi.op),
         ptr(pi.norms), ptr(pi.perm), pi.rows_pad, ni, f, pu.kp, pu.scale_exp, ptr(pu.row_exp), pi.scale_exp,
         ptr(_c(list_ids, I32)),
         ptr(_c(list_pos, I32)),
         ptr(_c(bounds, F64)), c, int(block),
         ptr(pb), ptr(pn), ptr(p_ids), ptr(p_ceil), b_pad, ptr(gq), ptr(perm), ptr(off), nq, k, ptr(ids), ptr(sc),
         ptr(vis), int(options),
         stream_ptr())
    return ids, sc, vis


def gemm_debug(pu: Packed, pi: Packed, f):
    out = torch.empty((pu.rows, pi.rows), dtype=torch.float32, device=pu.op.device)
    call("simdex_gemm_debug", ptr(pu.op), pu.rows, ptr(pi.op), pi.rows, f, pu.kp, ptr(out), stream_ptr())
    return out


def merge_topk(in_ids, in_scores, k_out):
    parts, nu, kk = in_ids.shape
    ids = torch.empty((nu, k_out), dtype=I32, device=in_ids.device)
    sc = torch.empty((nu, k_out), dtype=F64, device=in_ids.device)
    call("simdex_merge_topk", ptr(_c(in_ids, I32)), ptr(_c(in_scores, F64)), parts, nu, kk, k_out, ptr(ids),
         ptr(sc), stream_ptr())
    return ids, sc
