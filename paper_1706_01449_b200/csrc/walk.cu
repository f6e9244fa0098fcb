// The SimDex bounded list walk, Algorithm 1 (index.py:185-268,
// PAPER.md:662-687), one warp per query.
//
// Lanes score 32 consecutive list positions at once (float64, like the
// reference's dgemv at index.py:230); the chunk is then replayed in list order
// with two ballots: the first position whose ceiling the running K-th beats
// (stop, strict '>' as index.py:227) and the first position that would enter
// the running top-K under the (score desc, id asc) rule.  Only entering
// positions touch the top-K, which lives sorted in shared memory, so the
// result and the visited count are exactly the sequential ones.
#include <cfloat>

#include "common.cuh"

namespace simdex {
namespace {

struct WalkArgs {
  const double* users;
  const double* unorm;
  const double* items;
  int f;
  int64_t n;  // list length == number of items
  const int32_t* list_ids;
  const double* bounds;
  const int64_t* q_user;
  const int32_t* q_cluster;
  int64_t nq;
  int k_eff;
  int64_t start;
  const int32_t* warm_ids;
  const double* warm_scores;
  const int32_t* warm_count;
  int no_prune;
  int32_t* out_ids;
  double* out_scores;
  int64_t* out_visited;
  int warps_per_cta;
};

// Insert (s, id) into the sorted list (ts, ti) holding `cnt` entries, capacity k.
__device__ __forceinline__ void warp_insert(double* ts, int32_t* ti, int& cnt, int k, double s, int32_t id,
                                            int lane) {
  int before = 0;
  for (int i = lane; i < cnt; i += 32) before += ranks_before(ts[i], ti[i], s, id) ? 1 : 0;
  before = __reduce_add_sync(0xffffffffu, before);
  if (before >= k) return;  // does not enter (list full and ranks after the K-th)
  const int end = cnt < k ? cnt : k - 1;  // last index that moves is end-1 -> end
  for (int hi = end; hi > before; hi -= 32) {
    const int i = hi - 1 - lane;
    double vs = 0.0;
    int32_t vi = 0;
    const bool mv = i >= before;
    if (mv) {
      vs = ts[i];
      vi = ti[i];
    }
    __syncwarp();
    if (mv) {
      ts[i + 1] = vs;
      ti[i + 1] = vi;
    }
    __syncwarp();
  }
  if (lane == 0) {
    ts[before] = s;
    ti[before] = id;
  }
  __syncwarp();
  if (cnt < k) ++cnt;
}

__global__ void __launch_bounds__(256) walk_kernel(WalkArgs a) {
  extern __shared__ unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * a.warps_per_cta + w;
  const int k = a.k_eff;
  const size_t per_warp = (size_t)k * (sizeof(double) + sizeof(int32_t)) + (size_t)a.f * sizeof(double);
  unsigned char* base = smem + w * ((per_warp + 15) & ~size_t(15));
  double* us = reinterpret_cast<double*>(base);
  double* ts = us + a.f;
  int32_t* ti = reinterpret_cast<int32_t*>(ts + k);
  if (q >= a.nq) return;

  const int64_t urow = a.q_user[q];
  const int c = a.q_cluster[q];
  const double* u = a.users + urow * a.f;
  for (int i = lane; i < a.f; i += 32) us[i] = u[i];
  const double unorm = a.unorm[urow];
  const int32_t* L = a.list_ids + (int64_t)c * a.n;
  const double* B = a.bounds + (int64_t)c * a.n;

  int cnt = 0;
  int64_t j = 0;
  if (a.warm_count) {
    cnt = a.warm_count[q];
    for (int i = lane; i < cnt; i += 32) {
      ts[i] = a.warm_scores[q * k + i];
      ti[i] = a.warm_ids[q * k + i];
    }
    j = a.start;
  } else {
    j = a.start;
  }
  __syncwarp();
  int64_t visited = a.n;
  bool done = false;
  while (j < a.n && !done) {
    const int64_t pos = j + lane;
    const bool valid = pos < a.n;
    const int len = (a.n - j) < 32 ? (int)(a.n - j) : 32;
    double s = -DBL_MAX, ceil = DBL_MAX;
    int32_t id = INT32_MAX;
    if (valid) {
      id = L[pos];
      const double* x = a.items + (int64_t)id * a.f;
      double acc = 0.0;
      for (int t = 0; t < a.f; ++t) acc = fma(x[t], us[t], acc);
      s = acc;
      ceil = B[pos] * unorm;  // ceilings = list_bounds * ||u|| (index.py:205-206)
    }
    int p = 0;
    while (p < len) {
      if (cnt < k) {  // fill: the first k_eff positions enter unconditionally (index.py:217-223)
        const double sp = __shfl_sync(0xffffffffu, s, p);
        const int32_t ip = __shfl_sync(0xffffffffu, id, p);
        warp_insert(ts, ti, cnt, k, sp, ip, lane);
        ++p;
        continue;
      }
      const double m = ts[k - 1];
      const int32_t mi = ti[k - 1];
      const bool act = valid && lane >= p;
      const unsigned stop = a.no_prune ? 0u : __ballot_sync(0xffffffffu, act && m > ceil);
      const unsigned cand = __ballot_sync(0xffffffffu, act && ranks_before(s, id, m, mi));
      const int qs = stop ? __ffs(stop) - 1 : 32;
      const int qc = cand ? __ffs(cand) - 1 : 32;
      if (qs < 32 && qs <= qc) {
        visited = j + qs;
        done = true;
        break;
      }
      if (qc >= len) break;
      const double sq = __shfl_sync(0xffffffffu, s, qc);
      const int32_t iq = __shfl_sync(0xffffffffu, id, qc);
      warp_insert(ts, ti, cnt, k, sq, iq, lane);
      p = qc + 1;
    }
    j += len;
  }
  if (!done) visited = a.n;
  for (int i = lane; i < k; i += 32) {
    a.out_scores[q * k + i] = i < cnt ? ts[i] : -DBL_MAX;
    a.out_ids[q * k + i] = i < cnt ? ti[i] : -1;
  }
  if (lane == 0) a.out_visited[q] = visited;
}

__global__ void ws_visited_kernel(int64_t* visited, int64_t nq, int64_t block, int64_t n) {
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  // index.py:372-387: n when the prefix covers the list, else floored at B
  visited[q] = (block >= n) ? n : (visited[q] > block ? visited[q] : block);
}

}  // namespace

int launch_walk(const double* users, const double* user_norms, const double* items, int32_t f, int64_t ni,
                const int32_t* list_ids, const double* bounds, const int64_t* q_user, const int32_t* q_cluster,
                int64_t nq, int32_t k, int64_t start, const int32_t* warm_ids, const double* warm_scores,
                const int32_t* warm_count, int32_t no_prune, int32_t* out_ids, double* out_scores,
                int64_t* out_visited, cudaStream_t s) {
  if (nq == 0) return SIMDEX_OK;
  const int k_eff = (int)(k < ni ? k : ni);
  const size_t per_warp =
      (((size_t)k_eff * (sizeof(double) + sizeof(int32_t)) + (size_t)f * sizeof(double)) + 15) & ~size_t(15);
  const size_t budget = 200 * 1024;
  int wpc = (int)(budget / per_warp);
  if (wpc > 8) wpc = 8;
  if (wpc < 1) {
    set_error("simdex_walk: k=%d with f=%d exceeds the per-warp shared-memory top-K capacity", k, f);
    return SIMDEX_EUNSUPPORTED;
  }
  const size_t smem = per_warp * wpc;
  SIMDEX_CUDA(cudaFuncSetAttribute(walk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  WalkArgs a{users, user_norms, items, f, ni, list_ids, bounds, q_user, q_cluster, nq, k_eff, start,
             warm_ids, warm_scores, warm_count, no_prune, out_ids, out_scores, out_visited, wpc};
  walk_kernel<<<(unsigned)ceil_div(nq, wpc), 32 * wpc, smem, s>>>(a);
  SIMDEX_LAUNCH_CHECK("walk");
  return SIMDEX_OK;
}

int ws_fix_visited(int64_t* visited, int64_t nq, int64_t block, int64_t n, cudaStream_t s) {
  if (nq == 0) return SIMDEX_OK;
  ws_visited_kernel<<<(unsigned)ceil_div(nq, 256), 256, 0, s>>>(visited, nq, block, n);
  SIMDEX_LAUNCH_CHECK("ws_visited");
  return SIMDEX_OK;
}

}  // namespace simdex
