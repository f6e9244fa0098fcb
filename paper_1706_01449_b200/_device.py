"""Device residency of host factor matrices.

A FactorMatrix is immutable, so its device copies are computed once per
device and cached on the object: the float64 values (row-major, what the
exact kernels read), their row norms, and the packed fp16 tensor-core
operand.  Host->device copies go through pinned staging.
"""

from __future__ import annotations

import os
import warnings

import numpy as np
import torch

from . import _lib, _ops

# FactorMatrix values are read-only by contract; torch only ever reads them
warnings.filterwarnings("ignore", message="The given NumPy array is not writable")


def device():
    _lib.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


_SMALL_PAGEABLE = os.environ.get("SIMDEX_SMALL_PAGEABLE") == "1"  # A/B timing only


def to_device(a: np.ndarray, dtype=None) -> torch.Tensor:
    """Stream-ordered upload through pinned staging (torch's caching host
    allocator keeps the buffer until the copy has run).  A copy from pageable
    memory would synchronise the stream first, idling the GPU while the host
    queues the next launches, so even small arrays are staged."""
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    if t.numel() and (t.numel() * t.element_size() >= (1 << 20) or not _SMALL_PAGEABLE):
        t = t.pin_memory()
    return t.to(device(), non_blocking=True)


def _cache(matrix):
    dev = device()
    store = matrix.__dict__.setdefault("_device", {})
    return store.setdefault(dev.index, {})


def f64(matrix) -> torch.Tensor:
    c = _cache(matrix)
    if "f64" not in c:
        c["f64"] = to_device(matrix.values)
    return c["f64"]


def f32_exact(matrix):
    """float32 device copy when every value is exactly representable
    (BASELINE inputs are float32 upcast), else None."""
    c = _cache(matrix)
    if "f32" not in c:
        t, exact = _ops.to_f32(f64(matrix))
        c["f32"] = t if exact else None
    return c["f32"]


def packed(matrix) -> _ops.Packed:
    c = _cache(matrix)
    if "packed" not in c:
        x = f64(matrix)
        c["packed"] = _ops.pack(x, _ops.max_abs(x))
    return c["packed"]


def packed_users(matrix) -> _ops.Packed:
    """The user-side tensor-core operand: one power-of-two scale per row, so
    small-norm users keep the band of large ones (simdex_pack_f16_rows)."""
    c = _cache(matrix)
    if "packed_rows" not in c:
        if os.environ.get("SIMDEX_USER_SCALE") == "matrix":  # A/B: one matrix-wide scale
            c["packed_rows"] = packed(matrix)
        else:
            c["packed_rows"] = _ops.pack_rows(f64(matrix))
    return c["packed_rows"]


def packed_sorted(matrix) -> _ops.Packed:
    """The packed operand re-laid out by descending row norm (catalogue passes)."""
    c = _cache(matrix)
    if "packed_sorted" not in c:
        c["packed_sorted"] = _ops.norm_sorted(packed(matrix))
    return c["packed_sorted"]


def share_rows(parent, child, lo: int, hi: int) -> None:
    """Seed ``child``'s device cache (child = rows [lo, hi) of parent) with
    views of the parent's resident copies, so a shard costs no upload."""
    src = parent.__dict__.get("_device", {}).get(torch.cuda.current_device() if torch.cuda.is_available() else -1)
    if not src:
        return
    dst = _cache(child)
    if "f64" in src and "f64" not in dst:
        dst["f64"] = src["f64"][lo:hi]
    if "f32" in src and "f32" not in dst:
        dst["f32"] = None if src["f32"] is None else src["f32"][lo:hi]


def norms(matrix) -> torch.Tensor:
    c = _cache(matrix)
    if "packed_rows" in c:  # same norm arithmetic in both pack kernels
        return c["packed_rows"].norms
    return packed(matrix).norms


def drop(matrix):
    """Forget the device copies (e.g. to time host->device transfers)."""
    matrix.__dict__.get("_device", {}).clear()


_SIDE_STREAMS: dict = {}


def side_stream(dev) -> "torch.cuda.Stream":
    """One extra stream per device for copies that overlap the main stream's kernels."""
    s = _SIDE_STREAMS.get(dev.index)
    if s is None:
        s = _SIDE_STREAMS[dev.index] = torch.cuda.Stream(device=dev)
    return s


def to_host(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


def to_host_pinned(t: torch.Tensor) -> np.ndarray:
    """Device -> pinned host copy (DMA at full PCIe rate), returned as numpy."""
    if t.numel() * t.element_size() < (1 << 20):
        return t.cpu().numpy()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return h.numpy()


def to_host_pinned_many(*ts: torch.Tensor):
    """Several device -> pinned host copies behind one stream synchronisation."""
    outs = []
    for t in ts:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        outs.append(h)
    torch.cuda.current_stream().synchronize()
    return tuple(h.numpy() for h in outs)
