// The SimDex bounded list walk, Algorithm 1 (index.py:185-268,
// PAPER.md:662-687), one warp per query.
//
// A chunk is 32 consecutive list positions, scored in float64 (like the
// reference's dgemv at index.py:230) by 8-lane groups, four items per step:
// lane gl of a group keeps the user's factor pairs 2(gl + 8i), 2(gl + 8i)+1
// in registers and reads the same pairs of the item row, so every load of a
// group is one contiguous row segment (coalesced; exact float32 copies when
// the values allow, half the bytes), then a fixed-order xor reduction and a
// shuffle hand lane p the score of position j + p.  The chunk is replayed in list order
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
  const float* users32;  // exact float32 copies (both or neither) or null
  const float* items32;
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

template <int NV, class ET>
__global__ void __launch_bounds__(256) walk_kernel(WalkArgs a, const ET* __restrict__ users,
                                                   const ET* __restrict__ items) {
  extern __shared__ unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gl = lane & 7, grp = lane >> 3;
  const int k = a.k_eff;
  const int f = a.f;
  const bool pairs = (f & 1) == 0;
  const size_t per_warp = ((size_t)k * (sizeof(double) + sizeof(int32_t)) + 15) & ~size_t(15);
  unsigned char* base = smem + w * per_warp;
  double* ts = reinterpret_cast<double*>(base);
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
    // the user's factor pairs of this lane's group slot, in registers
    double u[2 * NV];
    const ET* ur = users + urow * (int64_t)f;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const int q = 2 * (gl + 8 * i);
      u[2 * i] = q < f ? (double)ur[q] : 0.0;
      u[2 * i + 1] = q + 1 < f ? (double)ur[q + 1] : 0.0;
    }
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
      int32_t id = valid ? L[pos] : INT32_MAX;
      const double ceil = valid ? B[pos] * unorm : DBL_MAX;  // ceilings = list_bounds * ||u|| (index.py:205-206)
      double s = -DBL_MAX;
#pragma unroll 2
      for (int st = 0; st < 8; ++st) {
        const int p = 4 * st + grp;  // chunk position this group scores in this step
        const int32_t idp = __shfl_sync(0xffffffffu, id, p);
        double d = 0.0;
        if (p < len) {
          const ET* x = items + (int64_t)idp * f;
#pragma unroll
          for (int i = 0; i < NV; ++i) {
            const int q = 2 * (gl + 8 * i);
            double x0 = 0.0, x1 = 0.0;
            if (q < f) {
              if (pairs) {
                if constexpr (sizeof(ET) == 4) {
                  const float2 v = *reinterpret_cast<const float2*>(x + q);
                  x0 = v.x;
                  x1 = v.y;
                } else {
                  const double2 v = *reinterpret_cast<const double2*>(x + q);
                  x0 = v.x;
                  x1 = v.y;
                }
              } else {
                x0 = (double)x[q];
                if (q + 1 < f) x1 = (double)x[q + 1];
              }
            }
            d = fma(x0, u[2 * i], d);
            d = fma(x1, u[2 * i + 1], d);
          }
        }
        d += __shfl_xor_sync(0xffffffffu, d, 4);
        d += __shfl_xor_sync(0xffffffffu, d, 2);
        d += __shfl_xor_sync(0xffffffffu, d, 1);
        const double got = __shfl_sync(0xffffffffu, d, 8 * (lane & 3));
        if ((lane >> 2) == st && valid) s = got;
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

// visited of a query answered by the exact scan instead of the walk (top-K
// too large for a warp's shared memory): Algorithm 1's stop position in
// closed form from the exact top-K ("visited"), one thread per
// query; the top-K items' list positions come from a linear scan of the list
// (a rare path: k beyond ~16k).
__global__ void walk_visited_closed_form_kernel(const int64_t* __restrict__ q_user, const int32_t* __restrict__ q_cluster,
                                                int64_t nq, const int32_t* __restrict__ list_ids,
                                                const double* __restrict__ bounds, const double* __restrict__ unorm,
                                                int64_t n, int k_eff, const int32_t* __restrict__ out_ids,
                                                const double* __restrict__ out_scores, int32_t* __restrict__ mark,
                                                int no_prune, int64_t* __restrict__ out_visited) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  if (no_prune) {
    out_visited[q] = n;
    return;
  }
  int32_t* mk = mark + q * ((n + 31) / 32);
  for (int t = 0; t < k_eff; ++t) {
    const int32_t id = out_ids[q * k_eff + t];
    if (id >= 0) atomicOr(&mk[id >> 5], 1 << (id & 31));
  }
  const int32_t* L = list_ids + (int64_t)q_cluster[q] * n;
  const double* B = bounds + (int64_t)q_cluster[q] * n;
  int64_t last = -1;
  for (int64_t j = 0; j < n; ++j) {
    const int32_t id = L[j];
    if (mk[id >> 5] & (1 << (id & 31))) last = j;
  }
  const double sk = out_scores[q * k_eff + k_eff - 1];
  const double un = unorm[q_user[q]];
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (B[mid] * un >= sk)
      lo = mid + 1;
    else
      hi = mid;
  }
  int64_t v = last + 1;
  if (v < k_eff) v = k_eff;
  if (v < lo) v = lo;
  out_visited[q] = v > n ? n : v;
}

template <int NV, class ET>
int launch_walk_kernel(const WalkArgs& a, const ET* users, const ET* items, int wpc, size_t smem, int64_t need,
                       cudaStream_t s) {
  static size_t set_for[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > set_for[dev & 15]) {
    SIMDEX_CUDA(cudaFuncSetAttribute(walk_kernel<NV, ET>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    set_for[dev & 15] = smem;
  }
  int occ = 0;
  SIMDEX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, walk_kernel<NV, ET>, 32 * wpc, smem));
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)occ * sm_count();
  if (grid > need) grid = need;
  ProfileScope _prof("walk", s);
  walk_kernel<NV, ET><<<(unsigned)grid, 32 * wpc, smem, s>>>(a, users, items);
  _prof.end();
  SIMDEX_LAUNCH_CHECK("walk");
  return SIMDEX_OK;
}

template <class ET>
int launch_walk_et(const WalkArgs& a, const ET* users, const ET* items, int wpc, size_t smem, int64_t need,
                   cudaStream_t s) {
  const int pairs = (a.f + 1) / 2;
  if (pairs <= 8) return launch_walk_kernel<1, ET>(a, users, items, wpc, smem, need, s);
  if (pairs <= 16) return launch_walk_kernel<2, ET>(a, users, items, wpc, smem, need, s);
  if (pairs <= 32) return launch_walk_kernel<4, ET>(a, users, items, wpc, smem, need, s);
  if (pairs <= 64) return launch_walk_kernel<8, ET>(a, users, items, wpc, smem, need, s);
  if (pairs <= 128) return launch_walk_kernel<16, ET>(a, users, items, wpc, smem, need, s);
  set_error("simdex_walk: f=%d above the register-resident user row (256)", a.f);
  return SIMDEX_EUNSUPPORTED;
}

}  // namespace

int launch_walk_tasks(const double* users, const double* unorm, const double* items, const float* users32,
                      const float* items32, int32_t f, int64_t n,
                      const int32_t* list_ids, const double* bounds, const int64_t* tasks, const int32_t* n_tasks_dev,
                      int64_t n_tasks_max, const int64_t* q_user, const int32_t* q_cluster, const int64_t* q_out,
                      int32_t k, int64_t start, const int32_t* warm_ids, const double* warm_scores,
                      const int32_t* warm_count, int32_t no_prune, int64_t ws_floor, int32_t* out_ids,
                      double* out_scores, int64_t* out_visited, cudaStream_t s) {
  if (n_tasks_max == 0) return SIMDEX_OK;
  const int k_eff = (int)(k < n ? k : n);
  const size_t per_warp = ((size_t)k_eff * (sizeof(double) + sizeof(int32_t)) + 15) & ~size_t(15);
  const size_t budget = 200 * 1024;
  int wpc = (int)(budget / per_warp);
  if (wpc > 8) wpc = 8;
  if (wpc < 1) {
    // the top-K does not fit a warp's shared memory: exact float64 scan of the
    // queried rows, visited from the closed form (start 0 walks only)
    if (start != 0 || tasks || q_out || warm_count) {
      set_error("simdex_walk: k=%d exceeds the per-warp top-K capacity for a warm-start walk", k);
      return SIMDEX_EUNSUPPORTED;
    }
    int rc = exact_topk_rows(users, items, n, f, q_user, n_tasks_max, k, out_ids, out_scores, s);
    if (rc) return rc;
    Scratch<int32_t> mark;
    SIMDEX_CUDA(mark.alloc((size_t)n_tasks_max * ((n + 31) / 32), s));
    SIMDEX_CUDA(cudaMemsetAsync(mark.p, 0, sizeof(int32_t) * n_tasks_max * ((n + 31) / 32), s));
    walk_visited_closed_form_kernel<<<(unsigned)ceil_div(n_tasks_max, 128), 128, 0, s>>>(
        q_user, q_cluster, n_tasks_max, list_ids, bounds, unorm, n, k_eff, out_ids, out_scores, mark.p, no_prune,
        out_visited);
    SIMDEX_LAUNCH_CHECK("walk_visited_closed_form");
    return SIMDEX_OK;
  }
  const size_t smem = per_warp * wpc;
  Scratch<unsigned long long> queue;
  SIMDEX_CUDA(queue.alloc(1, s));
  SIMDEX_CUDA(cudaMemsetAsync(queue.p, 0, sizeof(unsigned long long), s));
  WalkArgs a{users, unorm, items, users32, items32, f, n, list_ids, bounds, tasks, n_tasks_dev, n_tasks_max, q_user,
             q_cluster, q_out, k_eff, start, warm_ids, warm_scores, warm_count, no_prune, ws_floor, out_ids,
             out_scores, out_visited, wpc, queue.p};
  const int64_t need = ceil_div(n_tasks_max, wpc);
  if (users32 && items32) return launch_walk_et<float>(a, users32, items32, wpc, smem, need, s);
  return launch_walk_et<double>(a, users, items, wpc, smem, need, s);
}

int launch_walk(const double* users, const double* user_norms, const double* items, const float* users32,
                const float* items32, int32_t f, int64_t ni,
                const int32_t* list_ids, const double* bounds, const int64_t* q_user, const int32_t* q_cluster,
                int64_t nq, int32_t k, int64_t start, const int32_t* warm_ids, const double* warm_scores,
                const int32_t* warm_count, int32_t no_prune, int32_t* out_ids, double* out_scores,
                int64_t* out_visited, cudaStream_t s) {
  return launch_walk_tasks(users, user_norms, items, users32, items32, f, ni, list_ids, bounds, nullptr, nullptr, nq,
                           q_user, q_cluster, nullptr, k, start, warm_ids, warm_scores, warm_count, no_prune, -1,
                           out_ids, out_scores, out_visited, s);
}

}  // namespace simdex
