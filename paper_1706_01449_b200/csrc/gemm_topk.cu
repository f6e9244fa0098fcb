// Fused users x items tensor-core product + certified running top-K
// (brute.py:59-113 topk_matmul; the work-sharing prefix product of
// index.py:351-371).
//
// Persistent, warp-specialised sm_100a kernel.  A work unit is 256 users
// (two 128-row M tiles that share every item tile) against one item
// segment, streamed in 128-item N tiles:
//   warp 0      TMA producer: users tile once per unit, item tiles through a
//               multi-stage ring (128-byte swizzled, mbarrier complete_tx);
//   warp 1      MMA issuer: tcgen05.mma kind::f16 (bf16 x bf16 -> fp32) into
//               TMEM, 2 M tiles x 2 accumulator buffers x 128 columns = 512
//               columns, so the next tile's MMAs overlap this tile's epilogue;
//   warps 2..9  epilogue: one thread per user row, tcgen05.ld 32 columns at
//               a time, a chunk-max filter against the row's certified
//               threshold, and append of the rare surviving candidates.
//
// Certification (exactness from bf16): with operands rounded to bf16 (unit
// roundoff 2^-8, exactly scaled by powers of two) and fp32 accumulation,
// every approximate score v satisfies |v - s| <= e_j := eps*||u||*||i_j|| + e_abs
// with eps = 2^-7 + 2^-16 + (kp+16)*2^-22 + 2^-20 (representation, product and
// accumulation error, plus slack for the fp32 epilogue arithmetic).  Each row
// keeps candidates with hi = v + e_j >= T, where T is the k-th largest
// lo = v - e_j seen so far (a valid lower bound on the exact k-th score);
// items dropped or never kept have s <= hi < T <= s_k, so they cannot be in
// the exact top-k (not even by the id tie rule).  The survivors are rescored
// exactly in float64 and ordered (score desc, id asc) by the finalize kernel.
// A row whose band outgrows its buffer is flagged and recomputed by the exact
// float64 path.
#include <cuda.h>

#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "sm100.cuh"

namespace simdex {

int launch_walk_tasks(const double* users, const double* unorm, const double* items, int32_t f, int64_t n,
                      const int32_t* list_ids, const double* bounds, const int64_t* tasks, const int32_t* n_tasks_dev,
                      int64_t n_tasks_max, const int64_t* q_user, const int32_t* q_cluster, const int64_t* q_out,
                      int32_t k, int64_t start, const int32_t* warm_ids, const double* warm_scores,
                      const int32_t* warm_count, int32_t no_prune, int64_t ws_floor, int32_t* out_ids,
                      double* out_scores, int64_t* out_visited, cudaStream_t s);
int exact_topk_rows_mapped(const double* users, const double* items, int64_t ni, int32_t f, const int64_t* rows,
                           int64_t n_rows, int32_t k, const int64_t* out_map, int32_t* out_ids, double* out_scores,
                           cudaStream_t s);

namespace {
using namespace sm100;

constexpr int kUnitRows = 256;
constexpr int kTileM = 128;
constexpr int kTileN = 128;
constexpr int kSlab = kTileM * 128;  // one [128 rows x 64 bf16] swizzled slab: 16 KB
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr int kMaxCap = 512;
constexpr int kMaxKB = 4;  // kp <= 256
constexpr uint32_t kIdesc = idesc_bf16_f32(kTileM, kTileN);

struct Unit {
  int64_t a_row0;   // first packed user row (multiple of 256)
  int64_t b_row0;   // first item-operand row (multiple of 128)
  int32_t rows;     // valid user rows, 1..256
  int32_t n_items;  // valid item rows
};

struct TopkParams {
  const Unit* units;
  const int32_t* n_units;
  const float* item_nrm;     // [B rows] ||i|| 2^si rounded up (0 on padding)
  const float* item_nmax32;  // [B rows / 32]
  const float* row_cu;       // [A rows] eps ||u|| 2^su rounded up
  float e_abs;
  int kb;
  int k_steps;
  int stages;
  int cap;
  int k_eff;
  int32_t* cand_id;
  float* cand_lo;
  float* cand_hi;
  int32_t* row_count;
  int32_t* row_flags;
  int64_t* heap_ops;
  float* debug_out;
  int64_t debug_ld;
};

__device__ __forceinline__ void swapf(float& a, float& b) {
  float t = a;
  a = b;
  b = t;
}

// k-th largest (1-based) of a[0..n): three-way quickselect, a is permuted.
__device__ __noinline__ float kth_largest(float* a, int n, int k) {
  int lo = 0, hi = n - 1;
  const int want = k - 1;
  while (lo < hi) {
    const float pv = a[(lo + hi) >> 1];
    int lt = lo, i = lo, gt = hi;
    while (i <= gt) {
      if (a[i] > pv) {
        swapf(a[lt], a[i]);
        ++lt;
        ++i;
      } else if (a[i] < pv) {
        swapf(a[i], a[gt]);
        --gt;
      } else {
        ++i;
      }
    }
    if (want < lt)
      hi = lt - 1;
    else if (want > gt)
      lo = gt + 1;
    else
      return pv;
  }
  return a[lo];
}

// Raise T to the k-th largest lower bound in the buffer and drop every entry
// whose upper bound falls below it.
__device__ __noinline__ void compact_row(float* lo, float* hi, int32_t* id, int& cnt, float& T, int k_eff) {
  float tmp[kMaxCap];
  for (int e = 0; e < cnt; ++e) tmp[e] = lo[e];
  const float kth = kth_largest(tmp, cnt, k_eff);
  if (kth > T) T = kth;
  int w = 0;
  for (int e = 0; e < cnt; ++e) {
    if (hi[e] >= T) {
      lo[w] = lo[e];
      hi[w] = hi[e];
      id[w] = id[e];
      ++w;
    }
  }
  cnt = w;
}

__global__ void __launch_bounds__(kThreads, 1)
    gemm_topk_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const TopkParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int KB = p.kb, S = p.stages;
  uint8_t* a_sm = base;
  uint8_t* b_sm = base + 2 * KB * kSlab;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_sm + S * KB * kSlab);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* a_full = bars + 2 * S;
  uint64_t* a_empty = a_full + 1;
  uint64_t* t_full = a_full + 2;   // [2]
  uint64_t* t_empty = a_full + 4;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 6);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch(&map_a);
    tma_prefetch(&map_b);
    for (int s = 0; s < S; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(t_full + b, 1);
      mbar_init(t_empty + b, kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  const int n_units = *p.n_units;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int iter = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++iter) {
        const Unit un = p.units[u];
        const int ntile_a = un.rows > kTileM ? 2 : 1;
        if (iter > 0) mbar_wait(a_empty, (iter - 1) & 1);
        mbar_arrive_expect_tx(a_full, ntile_a * KB * kSlab);
        for (int h = 0; h < ntile_a; ++h)
          for (int kb = 0; kb < KB; ++kb)
            tma_load_2d(a_sm + (h * KB + kb) * kSlab, &map_a, a_full, kb * 64, (int)(un.a_row0 + h * kTileM));
        const int n_tiles = (un.n_items + kTileN - 1) / kTileN;
        for (int t = 0; t < n_tiles; ++t) {
          mbar_wait(empty + stage, phase ^ 1);
          mbar_arrive_expect_tx(full + stage, KB * kSlab);
          for (int kb = 0; kb < KB; ++kb)
            tma_load_2d(b_sm + (stage * KB + kb) * kSlab, &map_b, full + stage, kb * 64,
                        (int)(un.b_row0 + t * kTileN));
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      uint32_t acc = 0;
      int iter = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++iter) {
        const Unit un = p.units[u];
        const int ntile_a = un.rows > kTileM ? 2 : 1;
        mbar_wait(a_full, iter & 1);
        tc_fence_after();
        const int n_tiles = (un.n_items + kTileN - 1) / kTileN;
        for (int t = 0; t < n_tiles; ++t, ++acc) {
          const uint32_t buf = acc & 1, use = acc >> 1;
          mbar_wait(t_empty + buf, (use & 1) ^ 1);
          mbar_wait(full + stage, phase);
          tc_fence_after();
          for (int h = 0; h < ntile_a; ++h) {
            const uint32_t d = tbase + (buf * 2 + h) * kTileN;
            for (int ks = 0; ks < p.k_steps; ++ks) {
              const int kb = ks >> 2, kk = ks & 3;
              const uint64_t ad = umma_desc_sw128(smem_u32(a_sm + (h * KB + kb) * kSlab) + kk * 32);
              const uint64_t bd = umma_desc_sw128(smem_u32(b_sm + (stage * KB + kb) * kSlab) + kk * 32);
              mma_bf16(d, ad, bd, kIdesc, ks > 0 ? 1u : 0u);
            }
          }
          mma_commit(empty + stage);  // smem slot free once these MMAs retire
          mma_commit(t_full + buf);   // accumulators ready for the epilogue
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(a_empty);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;
    const int h = ew >> 2;         // M tile of this warp
    const int q = warp & 3;        // TMEM lane quarter this warp may access
    const int row_local = h * kTileM + q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint32_t acc = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const Unit un = p.units[u];
      const int ntile_a = un.rows > kTileM ? 2 : 1;
      const bool live = row_local < un.rows;
      const int64_t grow = un.a_row0 + row_local;
      const float cu = live ? p.row_cu[grow] : 0.f;
      float T = -INFINITY;
      int cnt = 0, flags = 0;
      int64_t hops = 0;
      int32_t* my_id = p.cand_id + grow * p.cap;
      float* my_lo = p.cand_lo + grow * p.cap;
      float* my_hi = p.cand_hi + grow * p.cap;
      const int n_tiles = (un.n_items + kTileN - 1) / kTileN;
      for (int t = 0; t < n_tiles; ++t, ++acc) {
        const uint32_t buf = acc & 1, use = acc >> 1;
        mbar_wait(t_full + buf, use & 1);
        tc_fence_after();
        if (h < ntile_a) {
          for (int ch = 0; ch < kTileN / 32; ++ch) {
            const int c0 = t * kTileN + ch * 32;
            const int nvalid = min(32, un.n_items - c0);
            if (nvalid <= 0) break;
            float v[32];
            tmem_ld32(tbase + lane_off + (buf * 2 + h) * kTileN + ch * 32, v);
            if (!live) continue;
            if (p.debug_out) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (i < nvalid) p.debug_out[grow * p.debug_ld + un.b_row0 + c0 + i] = v[i];
              continue;
            }
            if (flags) continue;
            float mx = -INFINITY;
#pragma unroll
            for (int i = 0; i < 32; ++i) mx = fmaxf(mx, i < nvalid ? v[i] : -INFINITY);
            const float nmax = __ldg(p.item_nmax32 + ((un.b_row0 + c0) >> 5));
            if (fmaf(cu, nmax, mx) + p.e_abs >= T) {
              const float* nrm = p.item_nrm + un.b_row0 + c0;
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                if (i < nvalid) {
                  const float e = fmaf(cu, __ldg(nrm + i), p.e_abs);
                  const float hi = v[i] + e;
                  if (hi >= T && !flags) {
                    my_lo[cnt] = v[i] - e;
                    my_hi[cnt] = hi;
                    my_id[cnt] = c0 + i;
                    ++cnt;
                    ++hops;
                    if (cnt == p.cap) {
                      compact_row(my_lo, my_hi, my_id, cnt, T, p.k_eff);
                      if (cnt > p.cap - max(8, p.cap / 8)) flags = 1;  // band wider than the buffer
                    }
                  }
                }
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(t_empty + buf);
      }
      if (live && h < ntile_a) {
        if (!flags && !p.debug_out && cnt > p.k_eff) compact_row(my_lo, my_hi, my_id, cnt, T, p.k_eff);
        p.row_count[grow] = cnt;
        p.row_flags[grow] = flags;
        if (p.heap_ops) p.heap_ops[grow] = hops;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, 512);
  }
}

// ---------------------------------------------------------------------------
// operand-side prep
// ---------------------------------------------------------------------------
__global__ void row_cu_kernel(const double* __restrict__ norms, int64_t rows, int64_t rows_pad, double scale,
                              float* __restrict__ cu) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows_pad) return;
  cu[r] = r < rows ? __double2float_ru(norms[r] * scale) : 0.f;
}

// per-row scaled norms (rounded up) + 32-row chunk maxima; one warp per chunk
__global__ void item_nrm_kernel(const double* __restrict__ norms, int64_t rows, int64_t rows_pad, double scale,
                                float* __restrict__ nrm, float* __restrict__ nmax32) {
  const int64_t chunk = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int64_t r = chunk * 32 + lane;
  if (chunk * 32 >= rows_pad) return;
  const float v = r < rows ? __double2float_ru(norms[r] * scale) : 0.f;
  nrm[r] = v;
  float m = v;
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) nmax32[chunk] = m;
}

// ---------------------------------------------------------------------------
// finalize: exact float64 rescoring of the certified candidates (warp per row)
// ---------------------------------------------------------------------------
struct FinalizeParams {
  int64_t total_rows;
  const int64_t* row_user;     // packed row -> user row (-1 = padding); null = identity (< nu)
  const int64_t* row_out;      // packed row -> output row; null = identity
  const int32_t* row_cluster;  // packed row -> cluster (work sharing); null = brute force
  int64_t nu;
  const double* users;
  const double* items;
  int f;
  const int32_t* list_ids;  // [C, n] (work sharing)
  const double* bounds;     // [C, n]
  const double* unorm;      // [nu]
  int64_t n;                // list length (= items)
  int64_t prefix;           // B' = min(B, n)
  int k_eff;
  int cap;
  const int32_t* cand_id;
  const int32_t* row_count;
  const int32_t* row_flags;
  int32_t* out_ids;
  double* out_scores;
  int64_t* out_visited;  // work sharing
  int32_t* warm_count;   // work sharing: entries held at B
  int64_t* walk_list;
  int32_t* walk_n;
  int64_t* over_list;
  int64_t* over_out;
  int32_t* over_n;
  int pow2;
};

__global__ void __launch_bounds__(256) finalize_kernel(const FinalizeParams p) {
  extern __shared__ unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t r = (int64_t)blockIdx.x * 8 + w;
  const size_t per_warp = ((size_t)p.pow2 * 12 + (size_t)p.f * 8 + 15) & ~size_t(15);
  unsigned char* mine = smem + w * per_warp;
  double* us = reinterpret_cast<double*>(mine);
  double* ss = us + p.f;
  int32_t* si = reinterpret_cast<int32_t*>(ss + p.pow2);
  if (r >= p.total_rows) return;
  const int64_t user = p.row_user ? p.row_user[r] : r;
  if (user < 0 || user >= p.nu) return;
  const int64_t out = p.row_out ? p.row_out[r] : r;
  const int c = p.row_cluster ? p.row_cluster[r] : 0;
  if (p.row_flags[r]) {
    if (lane == 0) {
      const int slot = atomicAdd(p.over_n, 1);
      p.over_list[slot] = p.row_cluster ? r : user;
      p.over_out[slot] = out;
    }
    return;
  }
  const int cnt = p.row_count[r];
  for (int i = lane; i < p.f; i += 32) us[i] = p.users[user * p.f + i];
  __syncwarp();
  const int32_t* cid = p.cand_id + r * p.cap;
  for (int e = lane; e < p.pow2; e += 32) {
    if (e < cnt) {
      const int32_t pos = cid[e];
      const int32_t item = p.row_cluster ? p.list_ids[(int64_t)c * p.n + pos] : pos;
      const double* x = p.items + (int64_t)item * p.f;
      double s = 0.0;
      for (int t = 0; t < p.f; ++t) s = fma(x[t], us[t], s);
      ss[e] = s;
      si[e] = item;
    } else {
      ss[e] = -DBL_MAX;
      si[e] = INT32_MAX;
    }
  }
  // warp bitonic sort by (score desc, id asc)
  for (int size = 2; size <= p.pow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncwarp();
      for (int i = lane; i < p.pow2 / 2; i += 32) {
        const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
        const bool up = (lo & size) == 0;
        const double a = ss[lo], b = ss[hi];
        const int32_t ia = si[lo], ib = si[hi];
        if (up ? ranks_before(b, ib, a, ia) : ranks_before(a, ia, b, ib)) {
          ss[lo] = b;
          ss[hi] = a;
          si[lo] = ib;
          si[hi] = ia;
        }
      }
    }
  }
  __syncwarp();
  const int held = cnt < p.k_eff ? cnt : p.k_eff;
  for (int i = lane; i < p.k_eff; i += 32) {
    p.out_ids[out * p.k_eff + i] = i < held ? si[i] : -1;
    p.out_scores[out * p.k_eff + i] = i < held ? ss[i] : -DBL_MAX;
  }
  if (p.row_cluster && lane == 0) {
    // index.py:372-387: the prefix covers the list -> n; K-th beats the next
    // ceiling -> B; otherwise continue the walk from B with this top-K.
    if (p.prefix >= p.n) {
      p.out_visited[out] = p.n;
    } else if (held == p.k_eff && ss[p.k_eff - 1] > p.bounds[(int64_t)c * p.n + p.prefix] * p.unorm[user]) {
      p.out_visited[out] = p.prefix;
    } else {
      p.warm_count[out] = held;
      p.walk_list[atomicAdd(p.walk_n, 1)] = r;
    }
  }
}

// ---------------------------------------------------------------------------
// work-sharing setup: grouped queries -> 256-aligned packed rows and units
// ---------------------------------------------------------------------------
// single CTA: per-cluster aligned offsets and the unit list
__global__ void ws_units_kernel(const int64_t* __restrict__ q_off, int c, int64_t b_pad, int64_t bp,
                                int64_t* __restrict__ a_off, Unit* __restrict__ units, int32_t* __restrict__ n_units) {
  if (threadIdx.x != 0) return;
  int64_t acc = 0;
  int nu = 0;
  for (int j = 0; j < c; ++j) {
    const int64_t cnt = q_off[j + 1] - q_off[j];
    a_off[j] = acc;
    for (int64_t r = 0; r < cnt; r += kUnitRows) {
      Unit un;
      un.a_row0 = acc + r;
      un.b_row0 = (int64_t)j * b_pad;
      un.rows = (int32_t)min((int64_t)kUnitRows, cnt - r);
      un.n_items = (int32_t)bp;
      units[nu++] = un;
    }
    acc += ((cnt + kUnitRows - 1) / kUnitRows) * kUnitRows;
  }
  a_off[c] = acc;
  *n_units = nu;
}

// packed row r of cluster j: user q_user[q_off[j] + (r - a_off[j])] or padding
__global__ void ws_rows_kernel(const int64_t* __restrict__ q_user, const int64_t* __restrict__ q_perm,
                               const int64_t* __restrict__ q_off, const int64_t* __restrict__ a_off, int c,
                               int64_t rows_max, const uint16_t* __restrict__ ub, int kp,
                               const float* __restrict__ u_cu, uint16_t* __restrict__ a_pk, float* __restrict__ cu,
                               int64_t* __restrict__ row_user, int64_t* __restrict__ row_out,
                               int32_t* __restrict__ row_cluster) {
  // one warp per packed row
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows_max || r >= a_off[c]) return;
  int lo = 0, hi = c - 1;  // last j with a_off[j] <= r
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (a_off[mid] <= r)
      lo = mid;
    else
      hi = mid - 1;
  }
  const int j = lo;
  const int64_t i = r - a_off[j];
  const bool live = i < q_off[j + 1] - q_off[j];
  const int64_t user = live ? q_user[q_off[j] + i] : -1;
  const uint4* src = reinterpret_cast<const uint4*>(ub + (live ? user : 0) * kp);
  uint4* dst = reinterpret_cast<uint4*>(a_pk + r * kp);
  for (int v = lane; v < kp / 8; v += 32) dst[v] = live ? src[v] : make_uint4(0, 0, 0, 0);
  if (lane == 0) {
    cu[r] = live ? u_cu[user] : 0.f;
    row_user[r] = user;
    row_out[r] = live ? (q_perm ? q_perm[q_off[j] + i] : q_off[j] + i) : -1;
    row_cluster[r] = j;
  }
}

__global__ void brute_units_kernel(int64_t nu, int64_t ni, Unit* units, int32_t* n_units) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nunits = (nu + kUnitRows - 1) / kUnitRows;
  if (u == 0) *n_units = (int32_t)nunits;
  if (u >= nunits) return;
  Unit un;
  un.a_row0 = u * kUnitRows;
  un.b_row0 = 0;
  un.rows = (int32_t)min((int64_t)kUnitRows, nu - u * kUnitRows);
  un.n_items = (int32_t)ni;
  units[u] = un;
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int make_map(CUtensorMap* m, const void* ptr, int64_t rows, int kp) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    SIMDEX_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return SIMDEX_EUNSUPPORTED;
    }
    fn = reinterpret_cast<EncodeTiledFn>(f);
  }
  cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kp * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld kp=%d", (int)r, (long long)rows, kp);
    return SIMDEX_ECUDA;
  }
  return SIMDEX_OK;
}

double eps_for(int kp) { return std::ldexp(1.0, -7) + std::ldexp(1.0, -16) + (kp + 16) * std::ldexp(1.0, -22) + std::ldexp(1.0, -20); }

int cap_for(int k_eff) {
  int c = 2 * k_eff + 32;
  int p = 64;
  while (p < c) p <<= 1;
  return p > kMaxCap ? kMaxCap : p;
}

struct GemmGeometry {
  int kb, stages;
  size_t smem;
};

int geometry(int kp, GemmGeometry* g) {
  g->kb = kp / 64;
  const size_t budget = 225 * 1024;
  const size_t fixed = 1024 + 2 * (size_t)g->kb * kSlab + 512;
  int s = 6;
  while (s > 1 && fixed + (size_t)s * g->kb * kSlab > budget) --s;
  g->stages = s;
  g->smem = fixed + (size_t)s * g->kb * kSlab;
  if (g->smem > budget) {
    set_error("feature dimension too large for the tensor-core path (kp=%d)", kp);
    return SIMDEX_EUNSUPPORTED;
  }
  return SIMDEX_OK;
}

int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const TopkParams& p, const GemmGeometry& g, int grid,
                cudaStream_t s) {
  SIMDEX_CUDA(cudaFuncSetAttribute(gemm_topk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
  gemm_topk_kernel<<<grid, kThreads, g.smem, s>>>(ma, mb, p);
  SIMDEX_LAUNCH_CHECK("gemm_topk");
  return SIMDEX_OK;
}

int finalize_smem(int pow2, int f, size_t* out) {
  const size_t per_warp = ((size_t)pow2 * 12 + (size_t)f * 8 + 15) & ~size_t(15);
  *out = per_warp * 8;
  if (*out > 200 * 1024) {
    set_error("finalize: candidate buffer too large");
    return SIMDEX_EUNSUPPORTED;
  }
  return SIMDEX_OK;
}

}  // namespace

// Brute-force fused path (topk_matmul).
int gemm_topk_brute(const double* users, const uint16_t* ub, const double* u_norm, int64_t nu, const double* items,
                    const uint16_t* ib, const double* i_norm, int64_t ni, int32_t f, int32_t kp, int32_t su,
                    int32_t si, int32_t k, int32_t* out_ids, double* out_scores, int64_t* heap_ops, float* debug_out,
                    cudaStream_t s) {
  const int k_eff = (int)(k < ni ? k : ni);
  GemmGeometry g;
  int rc = geometry(kp, &g);
  if (rc) return rc;
  const int64_t nu_pad = ceil_div(nu, 256) * 256, ni_pad = ceil_div(ni, 256) * 256;
  const int cap = cap_for(k_eff);
  const int64_t nunits = ceil_div(nu, kUnitRows);
  Scratch<Unit> units;
  Scratch<int32_t> n_units, cnt, flags, cid, over_n, walk_n;
  Scratch<float> lo, hi, cu, inrm, inmax;
  Scratch<int64_t> over_list, over_out;
  SIMDEX_CUDA(units.alloc(nunits, s));
  SIMDEX_CUDA(n_units.alloc(1, s));
  SIMDEX_CUDA(cnt.alloc(nu_pad, s));
  SIMDEX_CUDA(flags.alloc(nu_pad, s));
  SIMDEX_CUDA(cid.alloc((size_t)nu_pad * cap, s));
  SIMDEX_CUDA(lo.alloc((size_t)nu_pad * cap, s));
  SIMDEX_CUDA(hi.alloc((size_t)nu_pad * cap, s));
  SIMDEX_CUDA(cu.alloc(nu_pad, s));
  SIMDEX_CUDA(inrm.alloc(ni_pad, s));
  SIMDEX_CUDA(inmax.alloc(ni_pad / 32, s));
  SIMDEX_CUDA(over_n.alloc(1, s));
  SIMDEX_CUDA(walk_n.alloc(1, s));
  SIMDEX_CUDA(over_list.alloc(nu, s));
  SIMDEX_CUDA(over_out.alloc(nu, s));
  const double eps = eps_for(kp);
  brute_units_kernel<<<(unsigned)ceil_div(nunits, 256), 256, 0, s>>>(nu, ni, units.p, n_units.p);
  SIMDEX_LAUNCH_CHECK("brute_units");
  row_cu_kernel<<<(unsigned)ceil_div(nu_pad, 256), 256, 0, s>>>(u_norm, nu, nu_pad, eps * std::ldexp(1.0, su), cu.p);
  SIMDEX_LAUNCH_CHECK("row_cu");
  item_nrm_kernel<<<(unsigned)ceil_div(ni_pad / 32, 8), 256, 0, s>>>(i_norm, ni, ni_pad, std::ldexp(1.0, si), inrm.p,
                                                                      inmax.p);
  SIMDEX_LAUNCH_CHECK("item_nrm");
  CUtensorMap ma, mb;
  if ((rc = make_map(&ma, ub, nu_pad, kp))) return rc;
  if ((rc = make_map(&mb, ib, ni_pad, kp))) return rc;
  TopkParams p{};
  p.units = units.p;
  p.n_units = n_units.p;
  p.item_nrm = inrm.p;
  p.item_nmax32 = inmax.p;
  p.row_cu = cu.p;
  p.e_abs = (float)std::ldexp((double)(f + 1), -124);
  p.kb = g.kb;
  p.k_steps = (f + 15) / 16;
  p.stages = g.stages;
  p.cap = cap;
  p.k_eff = k_eff;
  p.cand_id = cid.p;
  p.cand_lo = lo.p;
  p.cand_hi = hi.p;
  p.row_count = cnt.p;
  p.row_flags = flags.p;
  p.heap_ops = heap_ops;
  p.debug_out = debug_out;
  p.debug_ld = ni;
  const int grid = (int)(nunits < sm_count() ? nunits : sm_count());
  if ((rc = launch_gemm(ma, mb, p, g, grid, s))) return rc;
  if (debug_out) return SIMDEX_OK;
  int pow2 = 1;
  while (pow2 < cap) pow2 <<= 1;
  size_t fsm;
  if ((rc = finalize_smem(pow2, f, &fsm))) return rc;
  SIMDEX_CUDA(cudaMemsetAsync(over_n.p, 0, sizeof(int32_t), s));
  FinalizeParams fp{};
  fp.total_rows = nu;
  fp.nu = nu;
  fp.users = users;
  fp.items = items;
  fp.f = f;
  fp.n = ni;
  fp.k_eff = k_eff;
  fp.cap = cap;
  fp.cand_id = cid.p;
  fp.row_count = cnt.p;
  fp.row_flags = flags.p;
  fp.out_ids = out_ids;
  fp.out_scores = out_scores;
  fp.over_list = over_list.p;
  fp.over_out = over_out.p;
  fp.over_n = over_n.p;
  fp.pow2 = pow2;
  SIMDEX_CUDA(cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
  finalize_kernel<<<(unsigned)ceil_div(nu, 8), 256, fsm, s>>>(fp);
  SIMDEX_LAUNCH_CHECK("finalize");
  int32_t n_over = 0;
  SIMDEX_CUDA(cudaMemcpyAsync(&n_over, over_n.p, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  SIMDEX_CUDA(cudaStreamSynchronize(s));
  if (n_over > 0)
    return exact_topk_rows_mapped(users, items, ni, f, over_list.p, n_over, k, over_out.p, out_ids, out_scores, s);
  return SIMDEX_OK;
}

// Work-sharing prefix path (query_batch with work sharing).
int gemm_topk_ws(const double* users, const uint16_t* ub, const double* unorm, int64_t nu, const double* items,
                 int64_t ni, int32_t f, int32_t kp, int32_t su, int32_t si, const int32_t* list_ids,
                 const double* bounds, int32_t c, int64_t block, const uint16_t* prefix_b, const double* prefix_norm,
                 int64_t b_pad, const int64_t* q_user, const int64_t* q_perm, const int64_t* q_off, int64_t nq,
                 int32_t k, int32_t* out_ids, double* out_scores, int64_t* out_visited, cudaStream_t s) {
  const int k_eff = (int)(k < ni ? k : ni);
  const int64_t bp = block < ni ? block : ni;
  GemmGeometry g;
  int rc = geometry(kp, &g);
  if (rc) return rc;
  const int64_t rows_max = nq + (int64_t)c * kUnitRows;
  const int64_t units_max = ceil_div(nq, kUnitRows) + c;
  const int cap = cap_for(k_eff);
  Scratch<Unit> units;
  Scratch<int32_t> n_units, cnt, flags, cid, over_n, walk_n, warm_cnt, rclus;
  Scratch<float> lo, hi, cu, ucu, inrm, inmax;
  Scratch<int64_t> a_off, row_user, row_out, walk_list, over_list, over_out;
  Scratch<uint16_t> a_pk;
  SIMDEX_CUDA(units.alloc(units_max, s));
  SIMDEX_CUDA(n_units.alloc(1, s));
  SIMDEX_CUDA(a_off.alloc(c + 1, s));
  SIMDEX_CUDA(a_pk.alloc((size_t)rows_max * kp, s));
  SIMDEX_CUDA(cu.alloc(rows_max, s));
  SIMDEX_CUDA(ucu.alloc(ceil_div(nu, 256) * 256, s));
  SIMDEX_CUDA(row_user.alloc(rows_max, s));
  SIMDEX_CUDA(row_out.alloc(rows_max, s));
  SIMDEX_CUDA(rclus.alloc(rows_max, s));
  SIMDEX_CUDA(cnt.alloc(rows_max, s));
  SIMDEX_CUDA(flags.alloc(rows_max, s));
  SIMDEX_CUDA(cid.alloc((size_t)rows_max * cap, s));
  SIMDEX_CUDA(lo.alloc((size_t)rows_max * cap, s));
  SIMDEX_CUDA(hi.alloc((size_t)rows_max * cap, s));
  SIMDEX_CUDA(inrm.alloc((size_t)c * b_pad, s));
  SIMDEX_CUDA(inmax.alloc((size_t)c * b_pad / 32, s));
  SIMDEX_CUDA(walk_list.alloc(rows_max, s));
  SIMDEX_CUDA(over_list.alloc(rows_max, s));
  SIMDEX_CUDA(over_out.alloc(rows_max, s));
  SIMDEX_CUDA(walk_n.alloc(1, s));
  SIMDEX_CUDA(over_n.alloc(1, s));
  SIMDEX_CUDA(warm_cnt.alloc(nq, s));
  const double eps = eps_for(kp);
  ws_units_kernel<<<1, 32, 0, s>>>(q_off, c, b_pad, bp, a_off.p, units.p, n_units.p);
  SIMDEX_LAUNCH_CHECK("ws_units");
  row_cu_kernel<<<(unsigned)ceil_div(nu, 256), 256, 0, s>>>(unorm, nu, nu, eps * std::ldexp(1.0, su), ucu.p);
  SIMDEX_LAUNCH_CHECK("row_cu");
  // rows past a_off[c] stay "padding" (row_user = -1) and are skipped by finalize
  SIMDEX_CUDA(cudaMemsetAsync(row_user.p, 0xff, sizeof(int64_t) * rows_max, s));
  ws_rows_kernel<<<(unsigned)ceil_div(rows_max, 8), 256, 0, s>>>(q_user, q_perm, q_off, a_off.p, c, rows_max, ub, kp,
                                                                   ucu.p, a_pk.p, cu.p, row_user.p, row_out.p,
                                                                   rclus.p);
  SIMDEX_LAUNCH_CHECK("ws_rows");
  item_nrm_kernel<<<(unsigned)ceil_div((int64_t)c * b_pad / 32, 8), 256, 0, s>>>(
      prefix_norm, (int64_t)c * b_pad, (int64_t)c * b_pad, std::ldexp(1.0, si), inrm.p, inmax.p);
  SIMDEX_LAUNCH_CHECK("item_nrm");
  CUtensorMap ma, mb;
  if ((rc = make_map(&ma, a_pk.p, rows_max, kp))) return rc;
  if ((rc = make_map(&mb, prefix_b, (int64_t)c * b_pad, kp))) return rc;
  TopkParams p{};
  p.units = units.p;
  p.n_units = n_units.p;
  p.item_nrm = inrm.p;
  p.item_nmax32 = inmax.p;
  p.row_cu = cu.p;
  p.e_abs = (float)std::ldexp((double)(f + 1), -124);
  p.kb = g.kb;
  p.k_steps = (f + 15) / 16;
  p.stages = g.stages;
  p.cap = cap;
  p.k_eff = k_eff;
  p.cand_id = cid.p;
  p.cand_lo = lo.p;
  p.cand_hi = hi.p;
  p.row_count = cnt.p;
  p.row_flags = flags.p;
  const int grid = (int)(units_max < sm_count() ? units_max : sm_count());
  if ((rc = launch_gemm(ma, mb, p, g, grid, s))) return rc;
  int pow2 = 1;
  while (pow2 < cap) pow2 <<= 1;
  size_t fsm;
  if ((rc = finalize_smem(pow2, f, &fsm))) return rc;
  SIMDEX_CUDA(cudaMemsetAsync(over_n.p, 0, sizeof(int32_t), s));
  SIMDEX_CUDA(cudaMemsetAsync(walk_n.p, 0, sizeof(int32_t), s));
  FinalizeParams fp{};
  fp.total_rows = rows_max;
  fp.row_user = row_user.p;
  fp.row_out = row_out.p;
  fp.row_cluster = rclus.p;
  fp.nu = nu;
  fp.users = users;
  fp.items = items;
  fp.f = f;
  fp.list_ids = list_ids;
  fp.bounds = bounds;
  fp.unorm = unorm;
  fp.n = ni;
  fp.prefix = bp;
  fp.k_eff = k_eff;
  fp.cap = cap;
  fp.cand_id = cid.p;
  fp.row_count = cnt.p;
  fp.row_flags = flags.p;
  fp.out_ids = out_ids;
  fp.out_scores = out_scores;
  fp.out_visited = out_visited;
  fp.warm_count = warm_cnt.p;
  fp.walk_list = walk_list.p;
  fp.walk_n = walk_n.p;
  fp.over_list = over_list.p;
  fp.over_out = over_out.p;
  fp.over_n = over_n.p;
  fp.pow2 = pow2;
  SIMDEX_CUDA(cudaFuncSetAttribute(finalize_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm));
  finalize_kernel<<<(unsigned)ceil_div(rows_max, 8), 256, fsm, s>>>(fp);
  SIMDEX_LAUNCH_CHECK("finalize");
  // continue from B with the warm top-K (index.py:376-387)
  rc = launch_walk_tasks(users, unorm, items, f, ni, list_ids, bounds, walk_list.p, walk_n.p, rows_max, row_user.p,
                         rclus.p, row_out.p, k, bp, out_ids, out_scores, warm_cnt.p, 0, -1, out_ids, out_scores,
                         out_visited, s);
  if (rc) return rc;
  // rows whose certified band overflowed: exact walk from 0, visited floored at B
  return launch_walk_tasks(users, unorm, items, f, ni, list_ids, bounds, over_list.p, over_n.p, rows_max, row_user.p,
                           rclus.p, row_out.p, k, 0, nullptr, nullptr, nullptr, 0, bp, out_ids, out_scores,
                           out_visited, s);
}

}  // namespace simdex
