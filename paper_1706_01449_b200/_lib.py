"""ctypes binding of the in-tree C-ABI library (include/simdex_b200.h).

The library is the product path: there is no CPU fallback.  Loading fails
loudly when the shared object is missing, and every device entry point raises
``RuntimeError`` when no CUDA device is visible.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SIMDEX_LIB_PATH") or os.path.join(_HERE, "lib", "libsimdex_b200.so")  # override: A/B timing only
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "simdex_b200.h")

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64

# name -> argtypes (all return int status except the two noted)
SIGNATURES = {
    "simdex_abi_version": [],
    "simdex_last_error": [],
    "simdex_launch_count": [],
    "simdex_profile_enable": [C.c_int],
    "simdex_profile_read": [C.c_char_p, P, P],
    "simdex_profile_reset": [],
    "simdex_device_info": [C.c_int, P, P, P],
    "simdex_ctx_create": [C.c_int, P],
    "simdex_ctx_destroy": [P],
    "simdex_ctx_set_query_token": [P, I64],
    "simdex_ctx_set_full_lists": [P, P, P, I64],
    "simdex_ctx_workspace_bytes": [P, P],
    "simdex_topk_exact": [P, I64, P, I64, I32, P, I64, I32, P, P, P],
    "simdex_max_abs": [P, I64, P, P],
    "simdex_pack_f16": [P, I64, I32, I32, I64, I32, P, P, P],
    "simdex_topk_matmul": [P, P, P, P, I64, P, P, P, P, P, I64, I64, I32, I32, I32, I32, I32, P, P, P, P],
    "simdex_pack_f16_rows": [P, I64, I32, I64, I32, P, P, P, P],
    "simdex_topk_matmul_ctx": [P, P, P, P, P, I64, P, P, P, P, P, I64, I64, I32, I32, I32, P, I32, I32, P, P, P, I32,
                               P],
    "simdex_norm_order": [P, I64, P, P],
    "simdex_to_f32": [P, I64, P, P, P],
    "simdex_kmeans_seed": [P, P, I64, I32, I32, I64, P, P, P, P, P],
    "simdex_kmeans_assign": [P, P, I64, I32, P, I32, P, P, P, P, P, P],
    "simdex_kmeans_update": [P, P, I64, I32, P, I32, P, P, P, P, P],
    "simdex_max_angles": [P, I64, I32, P, I32, P, P, P],
    "simdex_build_index": [P, I64, I32, P, P, I32, P, P, P, P, P],
    "simdex_list_positions": [P, I32, I64, P, P],
    "simdex_walk": [P, P, P, I32, I64, P, P, P, P, I64, I32, I64, P, P, P, I32, P, P, P, P],
    "simdex_walk32": [P, P, P, P, P, I32, I64, P, P, P, P, I64, I32, I64, P, P, P, I32, P, P, P, P],
    "simdex_query_ws": [P, P, P, P, I64, P, P, P, P, P, I64, I64, I32, I32, I32, I32, P, P, P, I32, I64, P, P, I64, P,
                        P, P, I64, I32, P, P, P, P],
    "simdex_query_ws_opts": [P, P, P, P, I64, P, P, P, P, P, I64, I64, I32, I32, I32, I32, P, P, P, I32, I64, P, P, I64,
                             P, P, P, I64, I32, P, P, P, I32, P],
    "simdex_query_ws_ctx": [P, P, P, P, P, I64, P, P, P, P, P, I64, I64, I32, I32, I32, P, I32, P, P, P, I32, I64, P,
                            P, P, P, I64, P, P, P, I64, I32, P, P, P, I32, P],
    "simdex_build_prefix_ordered": [P, P, I64, I32, P, I32, P, P, P, P, I32, I64, I64, P, P, P, P, P],
    "simdex_build_prefix_hybrid": [P, P, I64, I32, P, I32, P, P, P, P, I32, I64, I64, I64, P, P, P, P, P],
    "simdex_fallback_rows": [P],
    "simdex_executed_pairs": [P],
    "simdex_ws_stats": [P],
    "simdex_ctx_stats": [P, P],
    "simdex_group_queries": [P, I64, P, I32, P, P, P, P],
    "simdex_gemm_debug": [P, I64, P, I64, I32, I32, P, P],
    "simdex_build_prefix": [P, P, I64, I32, P, I32, I64, I64, P, P, P],
    "simdex_merge_topk": [P, P, I32, I64, I32, I32, P, P, P],
}

_lib = None
_lock = threading.Lock()


class SimdexError(RuntimeError):
    """A device-side failure reported by the C-ABI library."""


def load():
    """Load (once) and return the ctypes library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(make -C paper_1706_01449_b200/csrc).  There is no CPU fallback."
            )
        lib = C.CDLL(LIB_PATH)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = {"simdex_last_error": C.c_char_p, "simdex_launch_count": C.c_int64}.get(name, C.c_int)
        if lib.simdex_abi_version() != 1:
            raise ImportError("libsimdex_b200.so ABI version mismatch")
        _lib = lib
    return _lib


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_1706_01449_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback"
        )


def call(name, *args):
    """Invoke a C-ABI entry point, raising on a non-zero status."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.simdex_last_error().decode(errors="replace")
        raise SimdexError(f"{name} failed ({rc}): {msg}")


def launch_count() -> int:
    """Kernels launched by the library so far in this process."""
    return int(load().simdex_launch_count())


def profile(on: bool = True) -> None:
    """Record CUDA events around the library's main kernels (simdex_profile_*)."""
    call("simdex_profile_reset")
    call("simdex_profile_enable", 1 if on else 0)


def profile_read(name: str):
    """(total milliseconds, launches) recorded for kernel ``name``."""
    ms = C.c_double(0.0)
    n = C.c_int64(0)
    call("simdex_profile_read", name.encode(), C.byref(ms), C.byref(n))
    return ms.value, n.value


def ws_stats():
    """(queries, continued past B, B', n, f) of this thread's last work-sharing call."""
    buf = (C.c_int64 * 5)()
    call("simdex_ws_stats", C.cast(buf, C.c_void_p))
    return tuple(int(x) for x in buf)


def fallback_rows() -> int:
    """Rows of this thread's last serving call answered by the exact float64
    fallback (valid after the stream synchronised)."""
    out = C.c_int64(0)
    call("simdex_fallback_rows", C.byref(out))
    return out.value


def executed_pairs():
    """(user, item) pairs the tensor-core launches of this thread's last
    serving call multiplied: (first launch, second launch)."""
    buf = (C.c_int64 * 2)()
    call("simdex_executed_pairs", C.cast(buf, C.c_void_p))
    return int(buf[0]), int(buf[1])


class Context:
    """An execution context of its own (simdex_ctx_create): a workspace
    arena and statistic slots, for serving calls that run concurrently on
    different streams of one thread (the default context is per thread)."""

    def __init__(self, device: int | None = None):
        import torch
        self.handle = C.c_void_p()
        call("simdex_ctx_create", torch.cuda.current_device() if device is None else device, C.byref(self.handle))

    def stats(self):
        """(continued past B, band-overflow rows, pairs launch 1, pairs launch 2)
        of the last call on this context; valid once its stream synchronised."""
        buf = (C.c_int64 * 4)()
        call("simdex_ctx_stats", self.handle, C.cast(buf, C.c_void_p))
        return tuple(int(x) for x in buf)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and _lib is not None:
            try:
                _lib.simdex_ctx_destroy(h)
            except Exception:  # noqa: BLE001 -- interpreter shutdown
                pass



def workspace_bytes() -> int:
    """Arena size of this thread's default execution context on the current device."""
    out = C.c_int64(0)
    call("simdex_ctx_workspace_bytes", None, C.byref(out))
    return out.value


def ptr(t):
    """Raw device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return C.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def header_symbols(path=HEADER_PATH):
    """Every entry point declared in include/simdex_b200.h."""
    import re

    text = open(path).read()
    return sorted(set(re.findall(r"SIMDEX_API\s+(?:const\s+)?\w+\*?\s+(simdex_\w+)\s*\(", text)))
