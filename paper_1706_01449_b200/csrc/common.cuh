// Shared helpers for the SimDex B200 kernels: error state, launch checks,
// ordering predicates, and small warp utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <vector>

#include "../../include/simdex_b200.h"

namespace simdex {

void set_error(const char* fmt, ...);
int cuda_fail(cudaError_t e, const char* what);

#define SIMDEX_CHECK_ARG(cond, ...)        \
  do {                                     \
    if (!(cond)) {                         \
      ::simdex::set_error(__VA_ARGS__);    \
      return SIMDEX_EINVAL;                \
    }                                      \
  } while (0)

#define SIMDEX_CUDA(call)                                      \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return ::simdex::cuda_fail(_e, #call); \
  } while (0)

// same, inside internal helpers that return cudaError_t
#define SIMDEX_TRY(call)                 \
  do {                                   \
    cudaError_t _e = (call);             \
    if (_e != cudaSuccess) return _e;    \
  } while (0)

// Every kernel launch site ends with SIMDEX_LAUNCH_CHECK (or count_launches
// for loops), which also feeds simdex_launch_count().
void count_launches(int64_t n);
#define SIMDEX_LAUNCH_CHECK(name)      \
  do {                                 \
    ::simdex::count_launches(1);       \
    SIMDEX_CUDA(cudaGetLastError());   \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// RAII event pair around a kernel launch when simdex_profile_enable(1) is set.
class ProfileScope {
 public:
  ProfileScope(const char* name, cudaStream_t s);
  ~ProfileScope() { end(); }
  void end();

 private:
  std::string name_;
  cudaEvent_t a_ = nullptr, b_ = nullptr;
  cudaStream_t s_;
  bool on_ = false;
};

// Keep the device's stream-ordered pool warm: without this the pool returns
// freed scratch to the driver at every synchronisation and the next call pays
// for re-mapping it.
void keep_pool_warm();

// Stream-ordered scratch allocation (freed on the same stream).
template <class T>
struct Scratch {
  T* p = nullptr;
  cudaStream_t s = nullptr;
  cudaError_t alloc(size_t count, cudaStream_t stream) {
    keep_pool_warm();
    s = stream;
    if (count == 0) count = 1;
    return cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), stream);
  }
  ~Scratch() {
    if (p) cudaFreeAsync(p, s);
  }
};

int sm_count();

// ---------------------------------------------------------------------------
// Execution context (simdex_ctx_*): a device workspace arena reused across
// calls, so the serving entry points allocate nothing and never synchronise
// the host; a pinned host word per statistic; cross-stream ordering.  NULL
// in the C-ABI selects the calling thread's default context for the current
// device.  One call at a time per context (the default one is per thread).
// ---------------------------------------------------------------------------
struct Ctx;
Ctx* ctx_or_default(void* ctx);
// pinned host int64 slots of the context (valid after the stream synchronises)
int64_t* ctx_host_slots(Ctx* c);
// Reuse of a serving call's per-query-set setup (simdex_ctx_set_query_token):
// the caller's token for the query set served next on this context, and what
// the context's arena currently holds (token, arena generation, signature of
// the call's inputs); the arena generation changes whenever the arena moves.
struct CtxSetup {
  int64_t query_token = 0;
  int64_t held_token = 0;
  uint64_t held_gen = 0, held_sig = 0;
  // per-cluster full lists for the next work-sharing call (simdex_ctx_set_full_lists)
  const uint16_t* full_b = nullptr;
  const double* full_norm = nullptr;
  int64_t bf_pad = 0;
};
CtxSetup* ctx_setup(Ctx* c);
// fills out[0..n) with the squared norms of the n points (k-means assignment)
using P2Fill = int (*)(const void* points, int64_t n, int f, double* out, cudaStream_t s);
uint64_t ctx_arena_gen(Ctx* c);

// Typed buffers carved out of the context arena for ONE call: add() every
// buffer first, then commit() (grows the arena stream-ordered when needed,
// orders this stream after the context's previous stream, assigns pointers).
// The destructor records the end of the call for the next one's ordering.
class Workspace {
 public:
  Workspace(Ctx* c, cudaStream_t s);
  ~Workspace();
  template <class T>
  void add(T** p, size_t count) {
    reqs_.push_back(Req{reinterpret_cast<void**>(p), (count == 0 ? 1 : count) * sizeof(T)});
  }
  int commit();

 private:
  struct Req {
    void** p;
    size_t bytes;
  };
  Ctx* c_;
  cudaStream_t s_;
  std::vector<Req> reqs_;
  bool committed_ = false;
  bool capturing_ = false;
};

// ---------------------------------------------------------------------------
// Result ordering: (score desc, id asc)  -- index.py:158-163
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ bool ranks_before(double sa, int32_t ia, double sb, int32_t ib) {
  return sa > sb || (sa == sb && ia < ib);
}

// Orderable 64-bit key of a double so that ascending key == descending value,
// with -0.0 folded onto +0.0 (numpy compares them equal).
__host__ __device__ __forceinline__ uint64_t desc_key(double v) {
  if (v == 0.0) v = 0.0;
  uint64_t b;
  memcpy(&b, &v, 8);
  b = (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);  // ascending order
  return ~b;                                                           // descending
}

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int ceil_div_i(int a, int b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// internal entry points shared across translation units
// ---------------------------------------------------------------------------
// Batched (score desc, id asc) sort of `segs` equal-length segments of
// (key, id) pairs; keys are float64 values sorted descending.
cudaError_t segmented_sort_desc(double* keys, int32_t* ids, int64_t segs, int64_t len, cudaStream_t s);

// Positions 0..n-1 grouped by label assign[i] in [0, c), stable ((label,
// position) order), with counts [c] and offsets [c + 1] (kmeans.cu).
cudaError_t group_stable(const int64_t* assign, int64_t n, int c, int64_t* out_counts, int64_t* out_members,
                         int64_t* out_offsets, cudaStream_t s);

// Exact fp64 top-K of rows x a column set.  cols == nullptr means all ni
// items; otherwise cols[r] is a per-row... (not used).  Internal form used by
// topk_exact and by the overflow fallback of the tensor-core path.
int exact_topk_rows(const double* users, const double* items, int64_t ni, int32_t f,
                    const int64_t* rows, int64_t n_rows, int32_t k,
                    int32_t* out_ids, double* out_scores, cudaStream_t s);

int exact_topk_rows_mapped(const double* users, const double* items, int64_t ni, int32_t f, const int64_t* rows,
                           int64_t n_rows, int32_t k, const int64_t* out_map, int32_t* out_ids, double* out_scores,
                           cudaStream_t s);

// Exact float64 top-K of a DEVICE-counted row list (the band-overflow
// fallback of the tensor-core passes; no host round trip): for r < *n_rows,
// user row = user_of ? user_of[rows[r]] : rows[r], written to output row
// out_map[r].  `slab` is float64 [exact_slab_ctas(ni), ni] scratch.  k_eff <= 1024.
int exact_slab_ctas(int64_t ni);
int exact_topk_devcount(const double* users, const float* users32, const double* items, const float* items32,
                        int64_t ni, int32_t f, const int64_t* rows, const int64_t* user_of, const int32_t* n_rows,
                        int32_t k, const int64_t* out_map, int32_t* out_ids, double* out_scores, double* slab,
                        cudaStream_t s);

// Merge `parts` sorted lists per row.
int merge_lists(const int32_t* in_ids, const double* in_scores, int32_t parts, int64_t nu, int32_t kk,
                int32_t k_out, int32_t* out_ids, double* out_scores, cudaStream_t s);

}  // namespace simdex
