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
//
// The kernel is persistent: warps pull queries from an atomic work queue,
// which balances the very uneven walk lengths.  A query may start at a list
// position B with a warm top-K (work-sharing continuation, index.py:376-387).
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
  const int64_t* tasks;        // task -> query index (null: identity)
  const int32_t* n_tasks_dev;  // device task count (null: n_tasks)
  int64_t n_tasks;
  const int64_t* q_user;     // query -> user row
  const int32_t* q_cluster;  // query -> list row
  const int64_t* q_out;      // query -> output row (null: identity)
  int k_eff;
  int64_t start;
  const int32_t* warm_ids;  // [out rows, k_eff] (may alias out_ids)
  const double* warm_scores;
  const int32_t* warm_count;  // [out rows]
  int no_prune;
  int64_t ws_floor;  // >= 0: visited = max(visited, ws_floor)
  int32_t* out_ids;
  double* out_scores;
  int64_t* out_visited;
  int warps_per_cta;
  unsigned long long* queue;
};

// Insert (s, id) into the sorted list (ts, ti) holding `cnt` entries, capacity k.
__device__ __forceinline__ void warp_insert(double* ts, int32_t* ti, int& cnt, int k, double s, int32_t id,
                                            int lane) {
  int before = 0;
  for (int i = lane; i < cnt; i += 32) before += ranks_before(ts[i], ti[i], s, id) ? 1 : 0;
  before = __reduce_add_sync(0xffffffffu, before);
  if (before >= k) return;  // list full and (s, id) ranks after the K-th
  const int end = cnt < k ? cnt : k - 1;
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
  const int k = a.k_eff;
  const size_t per_warp = (((size_t)k * (sizeof(double) + sizeof(int32_t)) + (size_t)a.f * sizeof(double)) + 15) &
                          ~size_t(15);
  unsigned char* base = smem + w * per_warp;
  double* us = reinterpret_cast<double*>(base);
  double* ts = us + a.f;
  int32_t* ti = reinterpret_cast<int32_t*>(ts + k);
  const int64_t n_tasks = a.n_tasks_dev ? (int64_t)*a.n_tasks_dev : a.n_tasks;

  for (;;) {
    unsigned long long t = 0;
    if (lane == 0) t = atomicAdd(a.queue, 1ull);
    t = __shfl_sync(0xffffffffu, t, 0);
    if ((int64_t)t >= n_tasks) break;
    const int64_t qi = a.tasks ? a.tasks[t] : (int64_t)t;
    const int64_t out = a.q_out ? a.q_out[qi] : qi;
    const int64_t urow = a.q_user[qi];
    const int c = a.q_cluster[qi];
    const double* u = a.users + urow * a.f;
    for (int i = lane; i < a.f; i += 32) us[i] = u[i];
    const double unorm = a.unorm[urow];
    const int32_t* L = a.list_ids + (int64_t)c * a.n;
    const double* B = a.bounds + (int64_t)c * a.n;

    int cnt = 0;
    if (a.warm_count) {
      cnt = a.warm_count[out];
      for (int i = lane; i < cnt; i += 32) {
        ts[i] = a.warm_scores[out * k + i];
        ti[i] = a.warm_ids[out * k + i];
      }
    }
    int64_t j = a.start;
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
        for (int q = 0; q < a.f; ++q) acc = fma(x[q], us[q], acc);
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
    if (a.ws_floor >= 0 && visited < a.ws_floor) visited = a.ws_floor;
    __syncwarp();
    for (int i = lane; i < k; i += 32) {
      a.out_scores[out * k + i] = i < cnt ? ts[i] : -DBL_MAX;
      a.out_ids[out * k + i] = i < cnt ? ti[i] : -1;
    }
    if (lane == 0) a.out_visited[out] = visited;
    __syncwarp();
  }
}

}  // namespace

int launch_walk_tasks(const double* users, const double* unorm, const double* items, int32_t f, int64_t n,
                      const int32_t* list_ids, const double* bounds, const int64_t* tasks, const int32_t* n_tasks_dev,
                      int64_t n_tasks_max, const int64_t* q_user, const int32_t* q_cluster, const int64_t* q_out,
                      int32_t k, int64_t start, const int32_t* warm_ids, const double* warm_scores,
                      const int32_t* warm_count, int32_t no_prune, int64_t ws_floor, int32_t* out_ids,
                      double* out_scores, int64_t* out_visited, cudaStream_t s) {
  if (n_tasks_max == 0) return SIMDEX_OK;
  const int k_eff = (int)(k < n ? k : n);
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
  int occ = 0;
  SIMDEX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, walk_kernel, 32 * wpc, smem));
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)occ * sm_count();
  const int64_t need = ceil_div(n_tasks_max, wpc);
  if (grid > need) grid = need;
  Scratch<unsigned long long> queue;
  SIMDEX_CUDA(queue.alloc(1, s));
  SIMDEX_CUDA(cudaMemsetAsync(queue.p, 0, sizeof(unsigned long long), s));
  WalkArgs a{users, unorm, items, f, n, list_ids, bounds, tasks, n_tasks_dev, n_tasks_max, q_user, q_cluster, q_out,
             k_eff, start, warm_ids, warm_scores, warm_count, no_prune, ws_floor, out_ids, out_scores, out_visited,
             wpc, queue.p};
  ProfileScope _prof("walk", s);
  walk_kernel<<<(unsigned)grid, 32 * wpc, smem, s>>>(a);
  _prof.end();
  SIMDEX_LAUNCH_CHECK("walk");
  return SIMDEX_OK;
}

int launch_walk(const double* users, const double* user_norms, const double* items, int32_t f, int64_t ni,
                const int32_t* list_ids, const double* bounds, const int64_t* q_user, const int32_t* q_cluster,
                int64_t nq, int32_t k, int64_t start, const int32_t* warm_ids, const double* warm_scores,
                const int32_t* warm_count, int32_t no_prune, int32_t* out_ids, double* out_scores,
                int64_t* out_visited, cudaStream_t s) {
  return launch_walk_tasks(users, user_norms, items, f, ni, list_ids, bounds, nullptr, nullptr, nq, q_user, q_cluster,
                           nullptr, k, start, warm_ids, warm_scores, warm_count, no_prune, -1, out_ids, out_scores,
                           out_visited, s);
}

}  // namespace simdex
