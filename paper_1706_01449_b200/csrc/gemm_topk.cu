// Fused users x items tensor-core product + certified running top-K
// (brute.py:59-113 topk_matmul; the work-sharing product of index.py:351-371).
//
// Persistent, warp-specialised sm_100a kernel.  A work unit is 256 users
// (two 128-row M tiles that share every item tile) against one item
// segment, streamed in 128-item N tiles:
//   warp 0      TMA producer: users tile once per unit, item tiles through a
//               multi-stage ring (128-byte swizzled, mbarrier complete_tx);
//   warp 1      MMA issuer: tcgen05.mma kind::f16 (fp16 x fp16 -> fp32) into
//               TMEM, 2 M tiles x 2 accumulator buffers x 128 columns = 512
//               columns, so the next tile's MMAs overlap this tile's epilogue;
//   warps 2..9  epilogue: one thread per user row, tcgen05.ld 32 columns at
//               a time, a chunk-max filter against the row's certified
//               threshold, and append of the rare surviving candidates.
//
// Certification (exactness from fp16): with operands rounded to fp16 (unit
// roundoff 2^-11; scaled by exact powers of two so max|x| is in [1, 2)) and
// fp32 accumulation of the exact fp16 x fp16 products, every approximate
// score v satisfies |v - s| <= e_j := eps*||u||*||i_j|| + e_abs with
// eps = 2^-10 + 2^-22 + (kp+16)*2^-22 + 2^-20 (representation, accumulation,
// slack for the fp32 epilogue arithmetic) and e_abs = kp*2^-22 covering
// entries that land in fp16's subnormal range (absolute error <= 2^-25 each,
// |scaled entry| < 2).  Each row
// keeps candidates with hi = v + e_j >= T, where T is the k-th largest
// lo = v - e_j seen so far (a valid lower bound on the exact k-th score);
// items dropped or never kept have s <= hi < T <= s_k, so they cannot be in
// the exact top-k (not even by the id tie rule).  For k <= 32 the top-k of
// the lower bounds is held in registers (a branch-free insertion network), so
// T is always exact-current and the buffer only needs a linear filter; larger
// k keeps lower bounds in the buffer and re-selects T when it fills.  The
// survivors are rescored exactly in float64 and ordered (score desc, id asc)
// by the finalize kernel.  A row whose band outgrows its buffer is flagged and
// recomputed by the exact float64 path.
#include <cuda.h>

#include <cfloat>
#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include <cuda_fp16.h>

#include "common.cuh"
#include "sm100.cuh"

namespace simdex {

int exact_topk_rows_mapped(const double* users, const double* items, int64_t ni, int32_t f, const int64_t* rows,
                           int64_t n_rows, int32_t k, const int64_t* out_map, int32_t* out_ids, double* out_scores,
                           cudaStream_t s);

namespace {
using namespace sm100;

// mbarrier wait flavour per role (A/B builds): spinning try_wait, or try_wait
// with a suspend-time hint (the thread sleeps until the phase completes)
#ifndef SIMDEX_WAIT_PRODUCER
#define SIMDEX_WAIT_PRODUCER mbar_wait
#endif
#ifndef SIMDEX_WAIT_MMA
#define SIMDEX_WAIT_MMA mbar_wait
#endif

#ifndef SIMDEX_SPLIT_TARGET
#define SIMDEX_SPLIT_TARGET 8  // stage-2 units aimed at per CTA slot when catalogue segments are cut
#endif
#ifndef SIMDEX_LIST_STAGE2
#define SIMDEX_LIST_STAGE2 1
#endif
#ifndef SIMDEX_LIST_MIN_K
#define SIMDEX_LIST_MIN_K 8
#endif
#ifndef SIMDEX_LIST_MIN_Q
#define SIMDEX_LIST_MIN_Q 50000
#endif
#ifndef SIMDEX_M_TILES
#define SIMDEX_M_TILES 1
#endif
// finalize: two survivors per lane in one rescoring pass; resident CTAs per SM
// the register allocation is held to
#ifndef SIMDEX_FIN_TWO
#define SIMDEX_FIN_TWO 1
#endif
#ifndef SIMDEX_FIN_COOP
#define SIMDEX_FIN_COOP 1
#endif
#ifndef SIMDEX_FIN_ITEMS64
#define SIMDEX_FIN_ITEMS64 0
#endif
#ifndef SIMDEX_FIN_MINB
#define SIMDEX_FIN_MINB 5
#endif
// 128-row M tiles per unit and CTAs per SM: one M tile per CTA with two CTAs
// per SM (each CTA: 2 accumulator buffers x 128 columns of TMEM, 4 epilogue
// warps), so one CTA's slow epilogue warp never gates the other's hand-off
constexpr int kMTiles = SIMDEX_M_TILES;
constexpr int kCtasPerSm = kMTiles == 1 ? 2 : 1;
constexpr int kUnitRows = 128 * kMTiles;
constexpr int kTmemCols = kMTiles * 2 * 128;
constexpr int kTileM = 128;
constexpr int kTileN = 128;
constexpr int kSlab = kTileM * 128;  // one [128 rows x 64 fp16] swizzled slab: 16 KB
constexpr int kEpiWarps = 4 * kMTiles;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr int kMaxCap = 512;
constexpr uint32_t kIdesc = idesc_f16_f32(kTileM, kTileN);

struct Unit {
  int64_t a_row0;   // first packed user row (multiple of 256)
  int64_t b_row0;   // first item-operand row (multiple of 128)
  int64_t s_row0;   // first row of the per-row state (candidate buffers, counts, thresholds); a_row0
                    // except for catalogue segments of a split row block (their own state rows)
  int32_t rows;     // valid user rows, 1..256
  int32_t n_items;  // valid item rows
};

struct TopkParams {
  const Unit* units;
  const int32_t* n_units;
  const float* item_nrm;     // [B rows] ||i|| 2^si rounded up (0 on padding)
  const float* item_nmax32;  // [B rows / 32]
  const float* row_cu;       // [A rows] eps ||u|| 2^su rounded up
  const float* row_T0;       // [A rows] initial certified threshold (scaled domain) or null
  float e_abs;
  int kb;
  int k_steps;
  int stages;
  int cap;
  int k_eff;
  int32_t* cand_id;  // [A rows, cap]
  float* cand_lo;    // [A rows, cap] (k > 32 only)
  float* cand_hi;    // [A rows, cap]
  int32_t* row_count;
  int32_t* row_flags;
  float* row_T_out;  // [A rows] final certified threshold (finalize drops hi < T)
  int64_t* heap_ops;
  float* debug_out;
  int64_t debug_ld;
  int first_all;  // EXM = 2: a unit's first chunk stored whole with vector stores (list-order prefix)
  // item operand in descending-norm order: a unit stops streaming once no row
  // can take another candidate (Cauchy-Schwarz against the remaining norms)
  int norm_sorted;
  float g_mul;  // (1/eps + 2)(1 + 2^-20): ||u|| + 2 eps ||u|| from eps ||u|| (scaled, rounded up)
  float u_mul;  // (1/eps)(1 + 2^-20): ||u|| from eps ||u|| (scaled, rounded up)
  // per operand tile (global tile id = b_row0 / 128 + t), when given: every
  // item of tiles >= t of the unit's segment has score <= ||u|| exit_c and
  // norm <= exit_m (scaled); otherwise (norm-sorted operand) both are the
  // norm of the tile's first item
  const float* exit_c;
  const float* exit_m;
  unsigned long long* pairs_out;  // optional: (user row, item) pairs actually multiplied (valid rows x items)
};

#ifdef SIMDEX_EPI_TIMING
// diagnostic build only: clock64 cycle sums of CTA 0's warps 0 (producer),
// 1 (MMA), 2 (first epilogue warp), lane 0: [0] epilogue wait for full
// accumulators, [1] TMEM loads + wait, [2] tile processing, [3] tiles,
// [5] MMA wait for an empty accumulator buffer, [6] MMA wait for a full
// operand stage, [7] MMA tiles, [8] producer wait for an empty stage
__device__ unsigned long long g_epi_t[16];
#define EPI_T(i, v) atomicAdd(&g_epi_t[i], (unsigned long long)(v))
#endif
// three-input max (sm_100 FMNMX3)
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// k > 32, warp-cooperative: the 32 lanes jointly re-select lane `who`'s
// threshold T = k-th largest lower bound in its buffer (bitwise radix search
// over order-preserving keys, one warp-wide count per bit) and compact the
// buffer to the entries with hi >= T, preserving order.  Called with the whole
// warp converged; returns the new (cnt, T) of that lane.
__device__ __forceinline__ uint32_t f2key(float x) {
  const uint32_t b = __float_as_uint(x);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__device__ __noinline__ void warp_compact(float* lo, float* hi, int32_t* id, int cnt, int k_eff, float T_old,
                                          int lane, int* cnt_out, float* T_out) {
  constexpr int kPer = kMaxCap / 32;
  uint32_t key[kPer];
  float h[kPer];
  int32_t ids[kPer];
#pragma unroll
  for (int t = 0; t < kPer; ++t) {
    const int e = t * 32 + lane;
    key[t] = 0u;
    h[t] = -INFINITY;
    ids[t] = 0;
    if (e < cnt) {
      key[t] = f2key(lo[e]);
      h[t] = hi[e];
      ids[t] = id[e];
    }
  }
  uint32_t thr = 0;
  for (int b = 31; b >= 0; --b) {
    const uint32_t cand = thr | (1u << b);
    int c = 0;
#pragma unroll
    for (int t = 0; t < kPer; ++t) c += (t * 32 + lane < cnt && key[t] >= cand) ? 1 : 0;
    c = __reduce_add_sync(0xffffffffu, c);
    if (c >= k_eff) thr = cand;
  }
  float T = key2f(thr);
  if (T_old > T) T = T_old;
  __syncwarp();
  int w = 0;
#pragma unroll
  for (int t = 0; t < kPer; ++t) {
    const bool keep = (t * 32 + lane < cnt) && h[t] >= T;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int dst = w + __popc(m & ((1u << lane) - 1u));
      lo[dst] = key2f(key[t]);
      hi[dst] = h[t];
      id[dst] = ids[t];
    }
    w += __popc(m);
  }
  *cnt_out = w;
  *T_out = T;
}

// k <= 64, warp-cooperative: drop lane `who`'s buffer entries whose upper
// bound is below T, in place and order-preserving, 32 entries per step.
// Called with the whole warp converged; returns the new count.
__device__ __forceinline__ int warp_filter(float* hi, int32_t* id, int cnt, float T, int lane) {
  int w = 0;
  for (int base = 0; base < cnt; base += 32) {
    const int e = base + lane;
    float h = -INFINITY;
    int32_t i = 0;
    if (e < cnt) {
      h = hi[e];
      i = id[e];
    }
    const bool keep = e < cnt && h >= T;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    __syncwarp();
    if (keep) {  // destinations lie at or below this block: never a slot still to be read
      const int dst = w + __popc(m & ((1u << lane) - 1u));
      hi[dst] = h;
      id[dst] = i;
    }
    w += __popc(m);
    __syncwarp();
  }
  return w;
}

// sorted-descending top-KT insertion network: t <- top-KT of t + {x}
template <int KT>
__device__ __forceinline__ void push_top(float (&t)[KT], float x) {
#pragma unroll
  for (int i = KT - 1; i > 0; --i) t[i] = fmaxf(t[i], fminf(t[i - 1], x));
  t[0] = fmaxf(t[0], x);
}

template <int KT>
__device__ __forceinline__ float top_at(const float (&t)[KT], int k) {
  float r = t[0];
#pragma unroll
  for (int i = 1; i < KT; ++i) r = (i == k) ? t[i] : r;
  return r;
}

// EXM: early exit mode -- 0 none; 1 norm-sorted operand (the next tile's
// first norm bounds everything after it, checked every 4 tiles); 2 per-tile
// bound arrays exit_c / exit_m (the work-sharing prefix's list ceilings,
// checked after every tile)
template <int KT, int EXM>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    gemm_topk_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const TopkParams p) {
  constexpr bool EX = EXM != 0;
  constexpr int XM = EXM == 2 ? 0 : 3;  // exit checks / end markers at tiles t with (t & XM) == 0
  constexpr bool kDebug = KT < 0;         // raw accumulators to p.debug_out, no selection
  constexpr int KTT = KT > 0 ? KT : 1;    // register top-K size (KT = 0: buffer re-selection)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int KB = p.kb, S = p.stages;
  uint8_t* a_sm = base;
  uint8_t* b_sm = base + kMTiles * KB * kSlab;
  uint64_t* bars = reinterpret_cast<uint64_t*>(b_sm + S * KB * kSlab);
  uint64_t* full = bars;
  uint64_t* empty = bars + S;
  uint64_t* a_full = bars + 2 * S;
  uint64_t* a_empty = a_full + 1;
  uint64_t* t_full = a_full + 2;   // [2]
  uint64_t* t_empty = a_full + 4;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 6);
  // early-exit bookkeeping (norm-sorted operands), tagged so stale entries never match
  volatile int32_t* stage_end = reinterpret_cast<volatile int32_t*>(bars) + 64;   // [8] stage sequence no. of an end marker
  volatile int32_t* buf_end = stage_end + 8;                                      // [2] accumulator use no. of an end marker
  volatile long long* wdone = reinterpret_cast<volatile long long*>(bars) + 40;  // [8] (unit << 32) | tile after which a warp is done

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
    for (int i = 0; i < 8; ++i) {
      stage_end[i] = -1;
      wdone[i] = -1;
    }
    buf_end[0] = buf_end[1] = -1;
    for (int b = 0; b < 2; ++b) {
      mbar_init(t_full + b, 1);
      mbar_init(t_empty + b, kEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
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
      int32_t seq = 0;  // stages issued so far
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++iter) {
        const Unit un = p.units[u];
        const int ntile_a = un.rows > kTileM ? 2 : 1;
        if (iter > 0) SIMDEX_WAIT_PRODUCER(a_empty, (iter - 1) & 1);
        mbar_arrive_expect_tx(a_full, ntile_a * KB * kSlab);
        for (int h = 0; h < ntile_a; ++h)
          for (int kb = 0; kb < KB; ++kb)
            tma_load_2d(a_sm + (h * KB + kb) * kSlab, &map_a, a_full, kb * 64, (int)(un.a_row0 + h * kTileM));
        const int n_tiles = (un.n_items + kTileN - 1) / kTileN;
        for (int t = 0; t < n_tiles; ++t) {
          bool stop = EX && t > 0 && (t & XM) == 0;
          for (int w = 0; stop && w < kEpiWarps; ++w) {
            const long long e = wdone[w];
            stop = (int)(e >> 32) == u && (int)(e & 0xffffffffll) < t;
          }
#ifdef SIMDEX_EPI_TIMING
          const long long tp0 = clock64();
#endif
          SIMDEX_WAIT_PRODUCER(empty + stage, phase ^ 1);
#ifdef SIMDEX_EPI_TIMING
          if (blockIdx.x == 0) EPI_T(8, clock64() - tp0);
#endif
          if (stop) {  // every epilogue warp is done with this unit: end marker instead of tile t
            stage_end[stage] = seq;
            mbar_arrive(full + stage);
          } else {
            mbar_arrive_expect_tx(full + stage, KB * kSlab);
            for (int kb = 0; kb < KB; ++kb)
              tma_load_2d(b_sm + (stage * KB + kb) * kSlab, &map_b, full + stage, kb * 64,
                          (int)(un.b_row0 + t * kTileN));
          }
          ++seq;
          if (++stage == S) {
            stage = 0;
            phase ^= 1;
          }
          if (stop) break;
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
      // descriptors are built once: the start-address field (bits 0-13, in
      // 16-byte units) of a base descriptor is advanced by plain adds
      const uint64_t a_desc0 = umma_desc_sw128(smem_u32(a_sm));
      const uint64_t b_desc0 = umma_desc_sw128(smem_u32(b_sm));
      const int ksteps = p.k_steps;
      int32_t seq = 0;  // stages consumed so far
      unsigned long long pairs = 0;
      for (int u = blockIdx.x; u < n_units; u += gridDim.x, ++iter) {
        const Unit un = p.units[u];
        const int ntile_a = un.rows > kTileM ? 2 : 1;
        SIMDEX_WAIT_MMA(a_full, iter & 1);
        tc_fence_after();
        const int n_tiles = (un.n_items + kTileN - 1) / kTileN;
        for (int t = 0; t < n_tiles; ++t, ++acc) {
          const uint32_t buf = acc & 1, use = acc >> 1;
#ifdef SIMDEX_EPI_TIMING
          const long long tw0 = clock64();
#endif
          SIMDEX_WAIT_MMA(t_empty + buf, (use & 1) ^ 1);
#ifdef SIMDEX_EPI_TIMING
          const long long tw1 = clock64();
#endif
          SIMDEX_WAIT_MMA(full + stage, phase);
#ifdef SIMDEX_EPI_TIMING
          if (blockIdx.x == 0) {
            EPI_T(5, tw1 - tw0);
            EPI_T(6, clock64() - tw1);
            EPI_T(7, 1);
          }
#endif
          tc_fence_after();
          if (EX && (t & XM) == 0 && t > 0 && stage_end[stage] == seq) {  // end marker: pass it on to the epilogue
            mbar_arrive(empty + stage);
            buf_end[buf] = (int32_t)use;
            mbar_arrive(t_full + buf);
            ++seq;
            ++acc;
            if (++stage == S) {
              stage = 0;
              phase ^= 1;
            }
            break;
          }
          ++seq;
          pairs += (unsigned long long)un.rows * (unsigned long long)min(kTileN, un.n_items - t * kTileN);
          const uint64_t bd0 = b_desc0 + (uint64_t)((stage * KB * kSlab) >> 4);
          for (int h = 0; h < ntile_a; ++h) {
            const uint32_t d = tbase + (buf * kMTiles + h) * kTileN;
            const uint64_t ad0 = a_desc0 + (uint64_t)((h * KB * kSlab) >> 4);
#pragma unroll 4
            for (int ks = 0; ks < ksteps; ++ks) {
              const uint32_t off = (uint32_t)((ks >> 2) * (kSlab >> 4) + (ks & 3) * 2);
              mma_f16(d, ad0 + off, bd0 + off, kIdesc, ks > 0 ? 1u : 0u);
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
      if (p.pairs_out && pairs) atomicAdd(p.pairs_out, pairs);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int ew = warp - 2;
    const int h = ew >> 2;   // M tile of this warp
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row_local = h * kTileM + q * 32 + lane;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int kk = p.k_eff - 1;
    uint32_t acc = 0;
    for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
      const Unit un = p.units[u];
      const int ntile_a = un.rows > kTileM ? 2 : 1;
      const bool live = row_local < un.rows;
      const int64_t grow = un.a_row0 + row_local;
      const int64_t srow = un.s_row0 + row_local;  // this (row, catalogue segment)'s state
      const float cu = live ? p.row_cu[grow] : 0.f;
      float T = (live && p.row_T0) ? p.row_T0[grow] : -INFINITY;
      float top[KTT];
#pragma unroll
      for (int i = 0; i < KTT; ++i) top[i] = -INFINITY;
      int cnt = 0, flags = 0;
      int64_t hops = 0;
      int32_t* my_id = p.cand_id + srow * p.cap;
      float* my_lo = p.cand_lo + srow * p.cap;
      float* my_hi = p.cand_hi + srow * p.cap;
      const int n_tiles = (un.n_items + kTileN - 1) / kTileN;
      // the tile's four 32-item norm maxima, loaded one tile ahead (off the critical path)
      const float4* nm4p = reinterpret_cast<const float4*>(p.item_nmax32 + (un.b_row0 >> 5));
      float4 nm4_next = __ldg(nm4p);
      const float gu = cu * p.g_mul;  // ||u|| + 2 eps ||u||, scaled, rounded up
      const float uu = cu * p.u_mul;  // ||u||, scaled, rounded up
      const int64_t tile0 = un.b_row0 >> 7;
      float ec_next = 0.f, em_next = 0.f;
      if (EXM == 2 && n_tiles > 1) {
        ec_next = __ldg(p.exit_c + tile0 + 1);
        em_next = __ldg(p.exit_m + tile0 + 1);
      }
      bool done = false;              // no row of this warp can take another candidate
      for (int t = 0; t < n_tiles; ++t, ++acc) {
        const uint32_t buf = acc & 1, use = acc >> 1;
        const float4 nm4 = nm4_next;
        if (t + 1 < n_tiles) nm4_next = __ldg(nm4p + t + 1);
        const float ec = ec_next, em_ = em_next;  // bounds for the tiles after this one
        if (EXM == 2 && t + 2 < n_tiles) {
          ec_next = __ldg(p.exit_c + tile0 + t + 2);
          em_next = __ldg(p.exit_m + tile0 + t + 2);
        }
#ifdef SIMDEX_EPI_TIMING
        const bool tme = blockIdx.x == 0 && warp == 2 && lane == 0;
        const long long te0 = clock64();
        long long te_ld = 0;
#endif
        mbar_wait(t_full + buf, use & 1);
#ifdef SIMDEX_EPI_TIMING
        const long long te1 = clock64();
#endif
        tc_fence_after();
        if (EX && (t & XM) == 0 && t > 0 && buf_end[buf] == (int32_t)use) {  // the unit ended early
          __syncwarp();
          if (lane == 0) mbar_arrive(t_empty + buf);
          ++acc;
          break;
        }
        bool released = false;
        if (h < ntile_a && !(EX && done)) {
          const int tile_valid = min(kTileN, un.n_items - t * kTileN);
          // two chunks of 32 columns per TMEM wait; once the whole tile is in
          // registers the accumulator buffer goes back to the MMA warp
          constexpr int LDC = 2;
#pragma unroll
          for (int cg = 0; cg < kTileN / 32; cg += LDC) {
            if (cg * 32 >= tile_valid) break;
            uint32_t raw[LDC][32];
#pragma unroll
#ifdef SIMDEX_EPI_TIMING
            const long long tl0 = clock64();
#endif
            for (int c = 0; c < LDC; ++c)
              tmem_ld32_nowait(tbase + lane_off + (buf * kMTiles + h) * kTileN + (cg + c) * 32, raw[c]);
            tmem_wait_ld();
#ifdef SIMDEX_EPI_TIMING
            te_ld += clock64() - tl0;
#endif
            if (cg + LDC >= kTileN / 32) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(t_empty + buf);
              released = true;
            }
#pragma unroll
            for (int c = 0; c < LDC; ++c) {
              const int ch = cg + c;
              const int c0 = t * kTileN + ch * 32;
              const int nvalid = tile_valid - ch * 32;
              if (nvalid <= 0) break;
              if constexpr (kDebug) {
                if (live)
                  for (int i = 0; i < 32 && i < nvalid; ++i)
                    p.debug_out[grow * p.debug_ld + un.b_row0 + c0 + i] = __uint_as_float(raw[c][i]);
                continue;
              }
              float v[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(raw[c][i]);
              if (nvalid < 32) {  // the last, partial tile only (warp-uniform)
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = i < nvalid ? v[i] : -INFINITY;
              }
              // chunk max as a tree of 3-input FMNMX3 (17 instructions for 32 values)
              float m[11];
#pragma unroll
              for (int i = 0; i < 10; ++i) m[i] = fmax3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
              m[10] = fmaxf(v[30], v[31]);
              const float m0 = fmax3(m[0], m[1], m[2]), m1 = fmax3(m[3], m[4], m[5]);
              const float m2 = fmax3(m[6], m[7], m[8]), m3 = fmaxf(m[9], m[10]);
              const float mx = fmaxf(fmax3(m0, m1, m2), m3);
              const float nmax = ch == 0 ? nm4.x : ch == 1 ? nm4.y : ch == 2 ? nm4.z : nm4.w;
              const float em = fmaf(cu, nmax, p.e_abs);  // the chunk's widest band
              if constexpr (KT > 1) {
                // a unit's first chunk with no threshold yet (T = -inf in every
                // row): all 32 items go in with the chunk-wide band (hi = v + em
                // >= v + e_i, lo = v - em <= v - e_i: still certified bounds),
                // stored as vectors; the top-K of the lower bounds is built in
                // registers instead of 32 dependent append rounds
                if (t == 0 && ch == 0 && nvalid >= 32 &&
                    __all_sync(0xffffffffu, !(live && !flags) || (T == -INFINITY && cnt == 0))) {
                  if (live && !flags) {
#pragma unroll
                    for (int i = 0; i < 32; ++i) push_top<KTT>(top, v[i] - em);
                    T = fmaxf(T, KTT == kk + 1 ? top[KTT - 1] : top_at<KTT>(top, kk));
                    if (EXM == 2 && p.first_all) {
                      // prefix units that end within a few tiles: plain vector
                      // stores of all 32 (finalize drops those below T)
                      float4* dh = reinterpret_cast<float4*>(my_hi);
                      int4* di = reinterpret_cast<int4*>(my_id);
#pragma unroll
                      for (int q4 = 0; q4 < 8; ++q4) {
                        dh[q4] = make_float4(v[4 * q4] + em, v[4 * q4 + 1] + em, v[4 * q4 + 2] + em, v[4 * q4 + 3] + em);
                        di[q4] = make_int4(c0 + 4 * q4, c0 + 4 * q4 + 1, c0 + 4 * q4 + 2, c0 + 4 * q4 + 3);
                      }
                      cnt = 32;
                    } else {
                      // only the items that reach the new threshold are stored
                      // (compile-time register indices, a running store slot)
#pragma unroll
                      for (int i = 0; i < 32; ++i) {
                        const float hi = v[i] + em;
                        if (hi >= T) {
                          my_hi[cnt] = hi;
                          my_id[cnt] = c0 + i;
                          ++cnt;
                        }
                      }
                    }
                    hops += cnt;
                  }
                  continue;
                }
              }
              // rows that cannot take candidates (padding, overflowed) never pass
              const bool pass = mx + em >= ((live && !flags) ? T : INFINITY);
              // fast path: one vote per chunk; everything below is the rare, warp-uniform slow path
              if (!__any_sync(0xffffffffu, pass)) continue;
              const bool act = live && !flags;
              unsigned mask = 0;  // items of this chunk whose upper bound reaches T
              const float* nrm = p.item_nrm + un.b_row0 + c0;
              const float nrm_l = __ldg(nrm + lane);  // lane i holds item i's norm (coalesced)
              float vloc[32];  // the chunk, spilled for the appends: indexed dynamically
              if (pass) {
                if constexpr (KT == 1) {
                  // k = 1: the chunk max less the widest band lower-bounds its best item
                  top[0] = fmaxf(top[0], mx - em);
                  T = fmaxf(T, top[0]);
                }
                // coarse mask against the chunk-uniform band (a superset of the
                // per-item test, which the append loop applies): bit i set iff
                // v[i] - Tc >= 0, sign bits packed by funnel shifts
                const float Tc = (T - em) - fabsf(T) * 0x1p-22f - 0x1p-126f;
                unsigned neg = 0;
#pragma unroll
                for (int i = 31; i >= 0; --i) neg = __funnelshift_l(__float_as_uint(v[i] - Tc), neg, 1);
                mask = ~neg;
                if (nvalid < 32) mask &= (1u << nvalid) - 1u;  // -inf padding must not pass a -inf T
                if (mask) {
#pragma unroll
                  for (int i = 0; i < 32; ++i) vloc[i] = v[i];
                }
              }
              // converged append loop: every lane with pending items takes one per round
              while (__any_sync(0xffffffffu, mask != 0u)) {
                const int i = mask ? __ffs(mask) - 1 : 0;
                const float ni = __shfl_sync(0xffffffffu, nrm_l, i);  // item i's norm from lane i
                if (mask) {
                  mask &= mask - 1;
                  const float vi = vloc[i];
                  const float e = fmaf(cu, ni, p.e_abs);
                  const float hi = vi + e;
                  if (hi >= T && !flags) {  // T may have risen within this chunk
                    my_hi[cnt] = hi;
                    my_id[cnt] = c0 + i;
                    ++cnt;
                    ++hops;
                    if constexpr (KT > 0) {
                      push_top<KTT>(top, vi - e);
                      T = fmaxf(T, KTT == kk + 1 ? top[KTT - 1] : top_at<KTT>(top, kk));
                    } else {
                      my_lo[cnt - 1] = vi - e;  // the buffer always has >= 32 free slots here
                    }
                  }
                }
              }
              if constexpr (KT > 0) {
                // keep >= 32 free slots (a chunk appends at most 32): a nearly full
                // buffer is filtered against the current T by the whole warp
                unsigned full = __ballot_sync(0xffffffffu, cnt > p.cap - 32);
                while (full) {
                  const int who = __ffs(full) - 1;
                  full &= full - 1;
                  const int64_t g_w = __shfl_sync(0xffffffffu, srow, who);
                  const int c_w = __shfl_sync(0xffffffffu, cnt, who);
                  const float t_w = __shfl_sync(0xffffffffu, T, who);
                  const int nc = warp_filter(p.cand_hi + g_w * p.cap, p.cand_id + g_w * p.cap, c_w, t_w, lane);
                  if (lane == who) {
                    cnt = nc;
                    if (cnt > p.cap - 32 - max(8, p.cap / 8)) flags = 1;  // band wider than the buffer
                  }
                }
              }
              if constexpr (KT == 0) {
                // keep >= 32 free slots per row: re-select T for every full row, warp-cooperatively
                unsigned need = __ballot_sync(0xffffffffu, act && cnt > p.cap - 32);
                while (need) {
                  const int who = __ffs(need) - 1;
                  need &= need - 1;
                  const int64_t g_w = __shfl_sync(0xffffffffu, srow, who);
                  const int c_w = __shfl_sync(0xffffffffu, cnt, who);
                  const float t_w = __shfl_sync(0xffffffffu, T, who);
                  int nc;
                  float nt;
                  warp_compact(p.cand_lo + g_w * p.cap, p.cand_hi + g_w * p.cap, p.cand_id + g_w * p.cap, c_w,
                               p.k_eff, t_w, lane, &nc, &nt);
                  if (lane == who) {
                    cnt = nc;
                    T = nt;
                    if (cnt > p.cap - 32 - max(8, p.cap / 8)) flags = 1;  // band wider than the buffer
                  }
                }
              }
            }
          }
        }
        if (!released) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(t_empty + buf);
        }
#ifdef SIMDEX_EPI_TIMING
        if (tme) {
          const long long tproc = clock64() - te1 - te_ld;
          EPI_T(0, te1 - te0);
          EPI_T(1, te_ld);
          EPI_T(2, tproc);
          EPI_T(3, 1);
          // processing cycles by the tile's place in its unit: t = 0, 1-3, 4-7, >= 8
          EPI_T(9 + (t == 0 ? 0 : t < 4 ? 1 : t < 8 ? 2 : 3), tproc);
        }
#endif
        if (EX && !done && ((t + 1) & XM) == 0 && t + 1 < n_tiles) {
          // every later item has ||i|| <= the next tile's first norm, so its
          // upper bound is at most ||u|| n + 2 (eps ||u|| n + e_abs)
          const float bound = (EXM == 2 ? fmaf(uu, ec, 2.f * fmaf(cu, em_, p.e_abs))
                                        : fmaf(gu, nm4_next.x, 2.f * p.e_abs)) * (1.f + 0x1p-20f);
          if (__all_sync(0xffffffffu, !(live && !flags) || bound < T)) {
            done = true;
            if (lane == 0) wdone[ew] = ((long long)u << 32) | (long long)t;
          }
        }
      }
      if constexpr (KT == 0) {
        // final re-selection of T for every row of this warp (warp-cooperative)
        if (h < ntile_a) {
          unsigned need = __ballot_sync(0xffffffffu, live && !flags && cnt > p.k_eff);
          while (need) {
            const int who = __ffs(need) - 1;
            need &= need - 1;
            const int64_t g_w = __shfl_sync(0xffffffffu, srow, who);
            const int c_w = __shfl_sync(0xffffffffu, cnt, who);
            const float t_w = __shfl_sync(0xffffffffu, T, who);
            int nc;
            float nt;
            warp_compact(p.cand_lo + g_w * p.cap, p.cand_hi + g_w * p.cap, p.cand_id + g_w * p.cap, c_w, p.k_eff,
                         t_w, lane, &nc, &nt);
            if (lane == who) {
              cnt = nc;
              T = nt;
            }
          }
        }
      }
      if (live && h < ntile_a && !kDebug) {
        // the buffer may still hold entries admitted before T reached its final
        // value; finalize drops those against row_T_out in parallel
        p.row_count[srow] = cnt;
        p.row_flags[srow] = flags;
        p.row_T_out[srow] = T;
        if (p.heap_ops) p.heap_ops[srow] = hops;
      }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tbase, kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// operand-side prep
// ---------------------------------------------------------------------------
// cu[r] = eps ||u_r|| 2^(scale exponent of row r), rounded up; row_exp (per-row
// exponents of a simdex_pack_f16_rows operand) multiplies scale by 2^row_exp[r]
__global__ void row_cu_kernel(const double* __restrict__ norms, int64_t rows, int64_t rows_pad, double scale,
                              float* __restrict__ cu, const double* __restrict__ scale_dev = nullptr,
                              const int32_t* __restrict__ row_exp = nullptr) {
  int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows_pad) return;
  if (scale_dev) scale = *scale_dev;
  if (r < rows && row_exp) scale = ldexp(scale, row_exp[r]);
  cu[r] = r < rows ? __double2float_ru(norms[r] * scale) : 0.f;
}

// per-row scaled norms (rounded up) + 32-row chunk maxima; one warp per chunk
__global__ void item_nrm_kernel(const double* __restrict__ norms, int64_t rows, int64_t rows_pad, double scale,
                                float* __restrict__ nrm, float* __restrict__ nmax32,
                                const double* __restrict__ scale_dev = nullptr) {
  if (scale_dev) scale = *scale_dev;
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

// k-means assignment operands: argmin_j |p - c_j|^2 == argmax_j p'.c'_j with
// p' = [p, 1] and c' = [c, -|c|^2/2] (one extra K column, free while f < kp).
// Row norms for the certified band are guarded by alpha*(1 + |x|^2) per side:
// the product's cross term eps*alpha^2*(1+p2)(1+c2) >= 2^-39 (p2 + c2) covers
// the float64 rounding of d2 = (p2 + c2) - 2 p.c, so the exact float64 argmin
// is always among the candidates.
template <class P>
__global__ void max_abs_any_kernel(const P* __restrict__ x, int64_t n, double mul,
                                   unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs((double)x[i]) * mul);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// operand scales of the augmented product from the device maxima
// (m[0] = max|p|, m[1] = max|c|, m[2] = max |c|^2/2): exponents and the
// factors row_cu / item_nrm need -- no host round trip
__global__ void assign_scales_kernel(const unsigned long long* __restrict__ mx, double eps, int* __restrict__ sexp,
                                     double* __restrict__ sfac) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const double m0 = __longlong_as_double((long long)mx[0]), m1 = __longlong_as_double((long long)mx[1]),
               m2 = __longlong_as_double((long long)mx[2]);
  const double mu = fmax(m0, 1.0), mc = fmax(m1, m2);
  const int su = -ilogb(mu), sc = mc > 0.0 ? -ilogb(mc) : 0;
  sexp[0] = su;
  sexp[1] = sc;
  sfac[0] = eps * ldexp(1.0, su);
  sfac[1] = ldexp(1.0, sc);
}

// eight threads per row, each writing 16-byte pieces (8 halves) of the row
template <class P>
__global__ void pack_aug_kernel(const P* __restrict__ x, const double* __restrict__ sq, int64_t rows, int f,
                                int centers, const int* __restrict__ scale_exp_dev, int64_t rows_pad, int kp,
                                uint16_t* __restrict__ out, double* __restrict__ gnorm) {
  const int scale_exp = *scale_exp_dev;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r = g >> 3;
  const int sub = (int)(g & 7);
  if (r >= rows_pad) return;
  const bool live = r < rows;
  const double q = live ? sq[r] : 0.0;
  const double aug = live ? (centers ? -0.5 * q : 1.0) : 0.0;
  const double sc = ldexp(1.0, scale_exp);
  for (int k0 = sub * 8; k0 < kp; k0 += 64) {
    __align__(16) __half hv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int k = k0 + i;
      const double v = live ? (k < f ? (double)x[r * f + k] : (k == f ? aug : 0.0)) : 0.0;
      hv[i] = __double2half(v * sc);
    }
    *reinterpret_cast<uint4*>(out + r * kp + k0) = *reinterpret_cast<const uint4*>(hv);
  }
  if (sub == 0) gnorm[r] = live ? sqrt(q + aug * aug) * (1.0 + 0x1p-40) + 0x1p-16 * (1.0 + q) : 0.0;
}

// ---------------------------------------------------------------------------
// finalize: exact float64 rescoring of the certified candidates (warp per row)
// ---------------------------------------------------------------------------
enum FinalizeMode { kBrute = 0, kPrefix = 1, kFullList = 2, kAssign = 3 };

struct FinalizeParams {
  int mode;
  int64_t total_rows;
  const int32_t* n_rows_dev;   // device row count (stage 2); null: total_rows
  const int64_t* row_user;     // packed row -> user row (-1 = padding); null = identity (< nu)
  const int64_t* row_out;      // packed row -> output row; null = identity
  const int32_t* row_cluster;  // packed row -> cluster
  int64_t nu;
  const double* users;
  const double* items;
  const float* items32;     // exact float32 copy of items (half the bytes) or null
  int f;
  const int32_t* list_ids;  // [C, n]
  const int32_t* list_pos;  // [C, n] inverse of list_ids (full-list mode)
  const int32_t* item_perm; // item operand row -> item id (norm-sorted catalogue) or null
  const double* bounds;     // [C, n]
  const double* unorm;      // [nu]
  int64_t n;                // list length (= items)
  int64_t prefix;           // B' = min(B, n)
  int k_eff;
  int cap;
  const int32_t* cand_id;
  const float* cand_hi;   // upper bounds of the candidates (scaled domain)
  const float* row_T;     // final certified threshold per row (scaled domain)
  const int32_t* row_count;
  const int32_t* row_flags;
  int32_t* out_ids;
  double* out_scores;
  int64_t* out_visited;
  float* row_T0_out;   // prefix mode: certified lower bound for the full-list pass (scaled)
  double t0_scale;     // 2^(su+si)
  const int32_t* u_exp;  // per-user scale exponents (simdex_pack_f16_rows) or null: t0 also x 2^u_exp[user]
  const int32_t* prefix_ids;  // [C, prefix_ld] item id of each prefix operand row (reordered prefix) or null
  int64_t prefix_ld;
  int64_t* cont_list;  // prefix mode: rows that continue past B
  int32_t* cont_n;
  int64_t* over_list;
  int64_t* over_out;
  int32_t* over_n;
  int pow2;
  int coop;  // cooperative rescoring (finalize_coop())
  // list-order catalogue pass (full-list mode): candidate positions are list
  // positions from list_off on, and the row's prefix top-K (already in
  // out_ids, exact) joins the candidates; prefix rows whose band overflowed
  // go to the exact fallback list over1_* instead of continuing
  int64_t list_off;
  int merge_prefix;
  int64_t* over1_list;
  int64_t* over1_out;
  int32_t* over1_n;
  // k-means assignment mode (items = centers): d2 = (p2 + c2) - 2 p.c in
  // float64, first minimum over the certified candidates
  const float* users32;  // exact float32 copy of users or null
  const double* p2;
  const double* c2;
  const int64_t* prev;
  int64_t* out_assign;
  double* out_d2;
  unsigned long long* changed;
};

// First list position j with bounds[j] * unorm < s (ceilings are non-increasing).
__device__ int64_t ceiling_count(const double* b, int64_t n, double unorm, double s) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (b[mid] * unorm >= s)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// a row whose candidates do not fit: prefix rows redo the full list (stage
// 2 from T0 = -inf), other rows go to the exact float64 path
__device__ __forceinline__ void overflow_row(const FinalizeParams& p, int64_t r, int64_t user, int64_t out) {
  if (p.mode == kPrefix && p.over1_list) {  // list-order catalogue pass: the exact fallback takes the row
    const int sl = atomicAdd(p.over1_n, 1);
    p.over1_list[sl] = r;
    p.over1_out[sl] = out;
  } else if (p.mode == kPrefix) {
    p.row_T0_out[r] = -INFINITY;
    p.cont_list[atomicAdd(p.cont_n, 1)] = r;
  } else {
    const int sl = atomicAdd(p.over_n, 1);
    p.over_list[sl] = (p.mode == kBrute || p.mode == kAssign) ? user : r;
    p.over_out[sl] = out;
  }
}

#ifdef SIMDEX_EPI_TIMING
}  // namespace
extern "C" __attribute__((visibility("default"))) int simdex_dbg_epi_timing(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_epi_t, sizeof(g_epi_t));
  static const unsigned long long z[16] = {};
  return (int)cudaMemcpyToSymbol(g_epi_t, z, sizeof(z));
}
namespace {
#endif
#ifdef SIMDEX_FIN_STATS
// diagnostic build only: per finalize mode, sum over the rows' lanes of
// buffered candidates, of survivors of the final threshold, and of lanes
__device__ unsigned long long g_fin_stats[12];
}  // namespace
extern "C" __attribute__((visibility("default"))) int simdex_dbg_fin_stats(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_fin_stats, sizeof(g_fin_stats));
  static const unsigned long long z[12] = {};
  return (int)cudaMemcpyToSymbol(g_fin_stats, z, sizeof(z));
}
namespace {
#endif
// 4 rows per warp, 8 lanes per row: exact float64 rescoring of the row's
// certified candidates, (score desc, id asc) bitonic sort, output; plus the
// work-sharing bookkeeping of the mode.
// LPR lanes per row: 8 (4 rows per warp) for small k, 32 for k > 32
template <int LPR>
__global__ void __launch_bounds__(256, SIMDEX_FIN_MINB) finalize_kernel(const FinalizeParams p) {
  constexpr int RPW = 32 / LPR;
  extern __shared__ unsigned char smem[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int grp = lane / LPR, gl = lane % LPR;
  const unsigned gmask = LPR == 32 ? 0xffffffffu : (((1u << LPR) - 1u) << (grp * LPR));
  const int slot = w * RPW + grp;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) * RPW + slot;
  const size_t per_row = ((size_t)p.pow2 * 12 + (size_t)p.f * 8 + 15) & ~size_t(15);
  unsigned char* mine = smem + slot * per_row;
  // scores first (16-byte aligned rows: the rank loop and the rescoring read
  // pairs of doubles with one shared-memory load), then the user row, the ids
  double* ss = reinterpret_cast<double*>(mine);
  double* us = ss + p.pow2;
  int32_t* si = reinterpret_cast<int32_t*>(us + p.f);
  const int64_t total = p.n_rows_dev ? (int64_t)*p.n_rows_dev : p.total_rows;
  int64_t user = -1, out = -1;
  int c = 0, cnt = 0;
  bool act = false;
  if (r < total) {
    user = p.row_user ? p.row_user[r] : r;
    if (user >= 0 && user < p.nu) {
      out = p.row_out ? p.row_out[r] : r;
      c = (p.mode == kPrefix || p.mode == kFullList) ? p.row_cluster[r] : 0;
      if (p.row_flags[r]) {
        if (gl == 0) overflow_row(p, r, user, out);
      } else {
        act = true;
        cnt = p.row_count[r];
      }
    }
  }
  // warp-uniform loop bounds (the four rows share every warp instruction)
  const int cmax = __reduce_max_sync(0xffffffffu, cnt);
  if (__all_sync(0xffffffffu, !act)) return;
  int np2 = 2;
  while (np2 < cmax) np2 <<= 1;
  // cooperative rescoring (narrow rows, exact float32 copies): the 8 lanes of a
  // row share each candidate's item row -- every lane keeps its own factor
  // pairs of the user row in registers and reads the same pairs of the item
  // row, so a warp's gather touches 4 lines per load instead of up to 32 (the
  // kernel is bound by the L1 data pipe) -- and the 8 partial sums of a
  // candidate meet in the row's shared-memory block (the user row is not
  // staged there in this mode)
  const bool coop = SIMDEX_FIN_COOP && p.coop && LPR == 8 && p.mode != kAssign && p.items32 && p.users32 &&
                    (p.f & 1) == 0 && p.f <= 64 && p.f >= 36;
  if (act && !coop) {
    if (p.users32 && (p.f & 1) == 0) {  // two factors per load (rows of an even f are 8-byte aligned)
      const float2* u2 = reinterpret_cast<const float2*>(p.users32 + user * p.f);
      for (int i = gl; i < p.f / 2; i += LPR) {
        const float2 v = u2[i];
        *reinterpret_cast<double2*>(us + 2 * i) = make_double2((double)v.x, (double)v.y);
      }
    } else {
      for (int i = gl; i < p.f; i += LPR)
        us[i] = p.users32 ? (double)p.users32[user * p.f + i] : p.users[user * p.f + i];
    }
  }
  const int32_t* cid = p.cand_id + r * p.cap;
  const float* chi = p.cand_hi + r * p.cap;
  // keep the candidates whose upper bound reaches the row's final threshold
  // (compacted to the front in buffer order), resolve them to item ids
  const float Tr = act ? p.row_T[r] : 0.f;
  int kept = 0;
  for (int e0 = 0; e0 < cmax; e0 += LPR) {
    const int e = e0 + gl;
    const bool keep = act && e < cnt && chi[e] >= Tr;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const unsigned mine = (bal & gmask) >> (grp * LPR);
    if (keep) {
      const int dst = kept + __popc(mine & ((1u << gl) - 1u));
      if (dst < p.pow2) {
        const int32_t pos = cid[e];
        si[dst] = p.mode == kPrefix ? (p.prefix_ids ? p.prefix_ids[(int64_t)c * p.prefix_ld + pos]
                                                     : p.list_ids[(int64_t)c * p.n + pos])
                  : p.merge_prefix ? p.list_ids[(int64_t)c * p.n + p.list_off + pos]
                                   : (p.item_perm ? p.item_perm[pos] : pos);
      }
    }
    kept += __popc(mine);
  }
  if (p.merge_prefix) {
    // the prefix's exact top-K (positions < list_off, never among the
    // candidates) joins the rescoring
    for (int i0 = 0; i0 < p.k_eff; i0 += LPR) {
      const int i = i0 + gl;
      const int32_t id = (act && i < p.k_eff) ? p.out_ids[out * p.k_eff + i] : -1;
      const bool keep = id >= 0;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      const unsigned mine = (bal & gmask) >> (grp * LPR);
      if (keep) {
        const int dst = kept + __popc(mine & ((1u << gl) - 1u));
        if (dst < p.pow2) si[dst] = id;
      }
      kept += __popc(mine);
    }
  }
#ifdef SIMDEX_FIN_STATS
  if (act) {
    atomicAdd(&g_fin_stats[p.mode * 3], (unsigned long long)cnt);
    atomicAdd(&g_fin_stats[p.mode * 3 + 1], (unsigned long long)kept);
    atomicAdd(&g_fin_stats[p.mode * 3 + 2], 1ull);
  }
#endif
  if (act && kept > p.pow2) {  // more survivors than the row's shared-memory slots
    if (gl == 0) overflow_row(p, r, user, out);
    act = false;
    kept = 0;
  }
  cnt = kept;
  const int cmax2 = __reduce_max_sync(0xffffffffu, cnt);
  np2 = 2;
  while (np2 < cmax2) np2 <<= 1;
  __syncwarp();
  for (int e = cnt + gl; e < np2; e += LPR) {
    ss[e] = -DBL_MAX;
    si[e] = INT32_MAX;
  }
  __syncwarp();
  if (p.mode == kAssign) {
    // k-means: one lane per candidate, factors in order -- the arithmetic of
    // the squared norms, so a point equal to a centre gets exactly d2 = 0
    for (int e = gl; e < cmax2; e += LPR) {
      if (act && e < cnt) {
        double dot = 0.0;
        if (p.items32) {
          const float* x = p.items32 + (int64_t)si[e] * p.f;
          for (int q = 0; q < p.f; ++q) dot = fma((double)x[q], us[q], dot);
        } else {
          const double* x = p.items + (int64_t)si[e] * p.f;
          for (int q = 0; q < p.f; ++q) dot = fma(x[q], us[q], dot);
        }
        ss[e] = dot;
      }
    }
  }
  if (p.mode == kAssign) {  // clustering.py:100 + argmin (first minimum) over the candidates
    __syncwarp();
    double bd = DBL_MAX;
    int32_t bj = INT32_MAX;
    if (act) {
      const double pp = p.p2[user];
      for (int e = gl; e < cnt; e += LPR) {
        double d = (pp + p.c2[si[e]]) - 2.0 * ss[e];
        d = d > 0.0 ? d : 0.0;
        if (d < bd || (d == bd && si[e] < bj)) {
          bd = d;
          bj = si[e];
        }
      }
    }
    for (int o = LPR / 2; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int32_t oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (od < bd || (od == bd && oj < bj)) {
        bd = od;
        bj = oj;
      }
    }
    if (act && gl == 0) {
      p.out_assign[user] = bj;
      p.out_d2[user] = bd;
      if (p.prev && p.prev[user] != bj) atomicAdd(p.changed, 1ull);
    }
    return;
  }
  // exact float64 rescoring.  Narrow rows with several survivors per lane
  // group: one lane per candidate (two partial sums over the even / odd
  // factors, so identical rows still score identically); otherwise LPR/8
  // candidates per round, 8 lanes each (strided partials + xor tree)
  if (coop) {
    // this lane's factor pairs: float2 index v = 8 i + gl, i = 0..3
    // pairs 0..15 exist for every f >= 36; pairs 16 + gl and 24 + gl only below f / 2
    const int half = p.f >> 1;
    const bool ok2 = 16 + gl < half, ok3 = 24 + gl < half;
    const float2 zero2 = make_float2(0.f, 0.f);
    double2 uu[4];
    {
      const float2* ul = reinterpret_cast<const float2*>(p.users32) + (act ? user : 0) * half + gl;
      const float2 t0 = ul[0], t1 = ul[8], t2 = ok2 ? ul[16] : zero2, t3 = ok3 ? ul[24] : zero2;
      uu[0] = make_double2((double)t0.x, (double)t0.y);
      uu[1] = make_double2((double)t1.x, (double)t1.y);
      uu[2] = make_double2((double)t2.x, (double)t2.y);
      uu[3] = make_double2((double)t3.x, (double)t3.y);
    }
    const float2* items2 = reinterpret_cast<const float2*>(p.items32) + gl;
    double* part = us;  // [4 candidates][9]: 36 doubles of the (unused) user-row block
    for (int base = 0; base < cmax2; base += 4) {
#pragma unroll
      for (int c4 = 0; c4 < 4; ++c4) {
        const int e = base + c4;
        double a0 = 0.0, a1 = 0.0;
        if (act && e < cnt) {
          const float2* xl = items2 + (int64_t)si[e] * half;
          const float2 x0 = xl[0], x1 = xl[8], x2v = ok2 ? xl[16] : zero2, x3 = ok3 ? xl[24] : zero2;
          a0 = fma((double)x0.x, uu[0].x, a0);
          a1 = fma((double)x0.y, uu[0].y, a1);
          a0 = fma((double)x1.x, uu[1].x, a0);
          a1 = fma((double)x1.y, uu[1].y, a1);
          a0 = fma((double)x2v.x, uu[2].x, a0);
          a1 = fma((double)x2v.y, uu[2].y, a1);
          a0 = fma((double)x3.x, uu[3].x, a0);
          a1 = fma((double)x3.y, uu[3].y, a1);
        }
        part[c4 * 9 + gl] = a0 + a1;
      }
      __syncwarp();
      if (gl < 4) {  // lane c4 adds the candidate's 8 partials in lane order
        const int e = base + gl;
        if (act && e < cnt) {
          double t = part[gl * 9];
#pragma unroll
          for (int j = 1; j < 8; ++j) t += part[gl * 9 + j];
          ss[e] = t;
        }
      }
      __syncwarp();
    }
  }
  const bool lane_per_cand = !coop && p.f <= 64 && cmax2 > LPR / 2;
  constexpr int SG = LPR / 8;
  const int sg = gl >> 3, sl = gl & 7;
  for (int base = 0; base < (lane_per_cand || coop ? 0 : cmax2); base += SG) {
    const int e = base + sg;
    double part = 0.0;
    if (act && e < cnt) {
      if (p.items32) {
        const float* x = p.items32 + (int64_t)si[e] * p.f;
        for (int k0 = 0; k0 < p.f; k0 += 64) {
          float xv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) xv[i] = k0 + sl + 8 * i < p.f ? x[k0 + sl + 8 * i] : 0.f;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (k0 + sl + 8 * i < p.f) part = fma((double)xv[i], us[k0 + sl + 8 * i], part);
        }
      } else {
        const double* x = p.items + (int64_t)si[e] * p.f;
        for (int k0 = 0; k0 < p.f; k0 += 64) {
          double xv[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) xv[i] = k0 + sl + 8 * i < p.f ? x[k0 + sl + 8 * i] : 0.0;
#pragma unroll
          for (int i = 0; i < 8; ++i)
            if (k0 + sl + 8 * i < p.f) part = fma(xv[i], us[k0 + sl + 8 * i], part);
        }
      }
    }
    part += __shfl_xor_sync(0xffffffffu, part, 4);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    if (act && sl == 0 && e < cnt) ss[e] = part;
  }
  // up to two survivors per lane (the common case at K = 10: 9..16 per row):
  // one pass, the two candidates of a lane sharing the user-row loads; each
  // candidate's arithmetic is that of the single-candidate loop below
  const bool two_per_lane = SIMDEX_FIN_TWO && lane_per_cand && cmax2 > LPR && cmax2 <= 2 * LPR && p.items32 && (p.f & 1) == 0;
  if (two_per_lane) {
    const int e0 = gl, e1 = gl + LPR;
    if (act && e0 < cnt) {
      const bool has1 = e1 < cnt;
      const double2* u2 = reinterpret_cast<const double2*>(us);
      double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#if SIMDEX_FIN_ITEMS64
      // (A/B: the float64 item rows, twice the bytes, no conversions)
      const double2* xa = reinterpret_cast<const double2*>(p.items + (int64_t)si[e0] * p.f);
      const double2* xb = reinterpret_cast<const double2*>(p.items + (int64_t)si[has1 ? e1 : e0] * p.f);
#pragma unroll 5
      for (int q = 0; q < p.f / 2; ++q) {
        const double2 va = xa[q], vb = xb[q];
        const double2 u = u2[q];
        a0 = fma(va.x, u.x, a0);
        a1 = fma(va.y, u.y, a1);
        b0 = fma(vb.x, u.x, b0);
        b1 = fma(vb.y, u.y, b1);
      }
#else
      const float2* xa = reinterpret_cast<const float2*>(p.items32 + (int64_t)si[e0] * p.f);
      const float2* xb = reinterpret_cast<const float2*>(p.items32 + (int64_t)si[has1 ? e1 : e0] * p.f);
#pragma unroll 5
      for (int q = 0; q < p.f / 2; ++q) {
        const float2 va = xa[q], vb = xb[q];
        const double2 u = u2[q];
        a0 = fma((double)va.x, u.x, a0);
        a1 = fma((double)va.y, u.y, a1);
        b0 = fma((double)vb.x, u.x, b0);
        b1 = fma((double)vb.y, u.y, b1);
      }
#endif
      ss[e0] = a0 + a1;
      if (has1) ss[e1] = b0 + b1;
    }
  }
  for (int e = gl; e < (lane_per_cand && !two_per_lane ? cmax2 : 0); e += LPR) {
    if (act && e < cnt) {
      double d0 = 0.0, d1 = 0.0;
      const int64_t id = si[e];
      if (p.items32) {
        const float* x = p.items32 + id * p.f;
        if ((p.f & 1) == 0) {
          const float2* x2 = reinterpret_cast<const float2*>(x);
#pragma unroll 5
          for (int q = 0; q < p.f / 2; ++q) {
            const float2 v = x2[q];
            d0 = fma((double)v.x, us[2 * q], d0);
            d1 = fma((double)v.y, us[2 * q + 1], d1);
          }
        } else {
          for (int q = 0; q < p.f; ++q) d0 = fma((double)x[q], us[q], d0);
        }
      } else {
        const double* x = p.items + id * p.f;
        for (int q = 0; q < p.f; ++q) d0 = fma(x[q], us[q], d0);
      }
      ss[e] = d0 + d1;
    }
  }
  __syncwarp();
  const int held = act ? (cnt < p.k_eff ? cnt : p.k_eff) : 0;
  double kth = -DBL_MAX;
  int64_t mp = -1;
  if (cmax2 <= 32) {
    // few survivors: each candidate's rank under (score desc, id asc) is its
    // output slot.  Ranks are counted over the warp-uniform padded count:
    // slots [cnt, np2) hold (-DBL_MAX, INT32_MAX), which ranks before no
    // candidate.  A lane with two candidates (e, e + LPR) ranks both in one
    // pass over the slots.
    auto place = [&](int rank, double se, int32_t ie) {
      if (rank < p.k_eff) {
        p.out_ids[out * p.k_eff + rank] = ie;
        p.out_scores[out * p.k_eff + rank] = se;
        if (rank == p.k_eff - 1) kth = se;
        if (p.mode == kFullList) mp = max(mp, (int64_t)p.list_pos[(int64_t)c * p.n + ie]);
      }
    };
    if (cmax2 > LPR) {
      for (int e = gl; e < cmax2; e += 2 * LPR) {
        const int e1 = e + LPR;
        if (act && e < cnt) {
          const bool two = e1 < cnt;
          const double se0 = ss[e], se1 = two ? ss[e1] : se0;
          const int32_t ie0 = si[e], ie1 = two ? si[e1] : ie0;
          int rank0 = 0, rank1 = 0;
#pragma unroll 2
          for (int o = 0; o < np2; o += 2) {
            const double2 s2 = *reinterpret_cast<const double2*>(ss + o);
            const int2 i2 = *reinterpret_cast<const int2*>(si + o);
            rank0 += ranks_before(s2.x, i2.x, se0, ie0) ? 1 : 0;
            rank0 += ranks_before(s2.y, i2.y, se0, ie0) ? 1 : 0;
            rank1 += ranks_before(s2.x, i2.x, se1, ie1) ? 1 : 0;
            rank1 += ranks_before(s2.y, i2.y, se1, ie1) ? 1 : 0;
          }
          place(rank0, se0, ie0);
          if (two) place(rank1, se1, ie1);
        }
      }
    } else {
      const int e = gl;
      if (act && e < cnt) {
        const double se = ss[e];
        const int32_t ie = si[e];
        int rank = 0;
#pragma unroll 2
        for (int o = 0; o < np2; o += 2) {
          const double2 s2 = *reinterpret_cast<const double2*>(ss + o);
          const int2 i2 = *reinterpret_cast<const int2*>(si + o);
          rank += ranks_before(s2.x, i2.x, se, ie) ? 1 : 0;
          rank += ranks_before(s2.y, i2.y, se, ie) ? 1 : 0;
        }
        place(rank, se, ie);
      }
    }
    if (act)
      for (int i = held + gl; i < p.k_eff; i += LPR) {
        p.out_ids[out * p.k_eff + i] = -1;
        p.out_scores[out * p.k_eff + i] = -DBL_MAX;
      }
  } else {
    // bitonic sort by (score desc, id asc)
    for (int size = 2; size <= np2; size <<= 1) {
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        __syncwarp();
        for (int i = gl; i < np2 / 2; i += LPR) {
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
    if (act) {
      for (int i = gl; i < p.k_eff; i += LPR) {
        p.out_ids[out * p.k_eff + i] = i < held ? si[i] : -1;
        p.out_scores[out * p.k_eff + i] = i < held ? ss[i] : -DBL_MAX;
        if (p.mode == kFullList && i < held) mp = max(mp, (int64_t)p.list_pos[(int64_t)c * p.n + si[i]]);
      }
      if (held == p.k_eff) kth = ss[p.k_eff - 1];
    }
  }
  if (p.mode == kBrute) return;
  for (int o = LPR / 2; o > 0; o >>= 1) {
    kth = fmax(kth, __shfl_xor_sync(0xffffffffu, kth, o));
    mp = max(mp, __shfl_xor_sync(0xffffffffu, mp, o));
  }
  if (!act) return;
  if (p.mode == kPrefix) {
    // index.py:372-387: the prefix covers the list -> n; the K-th beats the
    // ceiling at B -> B; otherwise the user continues past B.
    bool cont = false;
    if (gl == 0) {
      if (p.prefix >= p.n) {
        p.out_visited[out] = p.n;
      } else if (held == p.k_eff && kth > p.bounds[(int64_t)c * p.n + p.prefix] * p.unorm[user]) {
        p.out_visited[out] = p.prefix;
      } else {
        // the prefix's exact K-th score lower-bounds the catalogue's: start the
        // full-list pass from it (rounded down, with a 2^-40 relative guard)
        float t0 = -INFINITY;
        if (held == p.k_eff) {
          const double sk = p.u_exp ? ldexp(kth * p.t0_scale, p.u_exp[user]) : kth * p.t0_scale;
          t0 = __double2float_rd(sk - fabs(sk) * 0x1p-40);
        }
        p.row_T0_out[r] = t0;
        cont = true;
      }
    }
    // one atomic per warp for the continuation list (not one per row)
    const unsigned am = __activemask();
    const unsigned cm = __ballot_sync(am, cont);
    if (cm) {
      const int leader = __ffs(cm) - 1;
      int base = 0;
      if (lane == leader) base = atomicAdd(p.cont_n, __popc(cm));
      base = __shfl_sync(am, base, leader);
      if (cont) p.cont_list[base + __popc(cm & ((1u << lane) - 1u))] = r;
    }
  }
  if (p.mode == kFullList) {
    // Exact top-K over the whole list is known, so Algorithm 1's sequential
    // stop position follows in closed form ("visited"): with P =
    // 1 + the largest list position of a top-K item and s_K the K-th score,
    //   visited = min(n, max(P, k_eff, #{j : bounds[j]*||u|| >= s_K})),
    // floored at B for work sharing (index.py:372-387).
    if (gl == 0) {
      const int64_t q = ceiling_count(p.bounds + (int64_t)c * p.n, p.n, p.unorm[user], kth);
      int64_t v = max(max(mp + 1, (int64_t)p.k_eff), q);
      if (v > p.n) v = p.n;
      if (v < p.prefix) v = p.prefix;
      p.out_visited[out] = v;
    }
  }
}

// visited for rows the exact fallback handled on the full list (same closed form)
__global__ void fallback_visited_kernel(const int64_t* __restrict__ rows, const int32_t* n_rows,
                                        const int64_t* __restrict__ row_user, const int64_t* __restrict__ row_out,
                                        const int32_t* __restrict__ row_cluster, const int32_t* __restrict__ list_pos,
                                        const double* __restrict__ bounds, const double* __restrict__ unorm, int64_t n,
                                        int64_t prefix, int k_eff, const int32_t* __restrict__ out_ids,
                                        const double* __restrict__ out_scores, int64_t* __restrict__ out_visited) {
  const int64_t cnt = *n_rows;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = rows[i];
    const int64_t user = row_user[r], out = row_out[r];
    const int c = row_cluster[r];
    int64_t mp = -1;
    for (int t = 0; t < k_eff; ++t) mp = max(mp, (int64_t)list_pos[(int64_t)c * n + out_ids[out * k_eff + t]]);
    const int64_t q = ceiling_count(bounds + (int64_t)c * n, n, unorm[user], out_scores[out * k_eff + k_eff - 1]);
    int64_t v = max(max(mp + 1, (int64_t)k_eff), q);
    if (v > n) v = n;
    if (v < prefix) v = prefix;
    out_visited[out] = v;
  }
}

// ---------------------------------------------------------------------------
// work-sharing setup
// ---------------------------------------------------------------------------
// one CTA (1024 threads): per-cluster 256-aligned row offsets and the unit
// list; thread t owns a contiguous run of clusters, runs are scanned in order
__global__ void __launch_bounds__(1024) ws_units_kernel(const int64_t* __restrict__ q_off, int c, int64_t b_pad,
                                                        int64_t bp, int64_t* __restrict__ a_off,
                                                        Unit* __restrict__ units, int32_t* __restrict__ n_units,
                                                        int64_t b_off = 0, int32_t* __restrict__ rows_out = nullptr) {
  __shared__ int64_t s_rows[1024];
  __shared__ int s_units[1024];
  const int t = threadIdx.x;
  const int per = (c + 1023) / 1024;
  const int j0 = min(c, t * per), j1 = min(c, j0 + per);
  int64_t rows = 0;
  int nun = 0;
  for (int j = j0; j < j1; ++j) {
    const int64_t cnt = q_off[j + 1] - q_off[j];
    const int64_t u = (cnt + kUnitRows - 1) / kUnitRows;
    rows += u * kUnitRows;
    nun += (int)u;
  }
  s_rows[t] = rows;
  s_units[t] = nun;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele scan
    const int64_t r2 = t >= off ? s_rows[t - off] : 0;
    const int u2 = t >= off ? s_units[t - off] : 0;
    __syncthreads();
    s_rows[t] += r2;
    s_units[t] += u2;
    __syncthreads();
  }
  int64_t acc = s_rows[t] - rows;
  int nu = s_units[t] - nun;
  for (int j = j0; j < j1; ++j) {
    const int64_t cnt = q_off[j + 1] - q_off[j];
    a_off[j] = acc;
    for (int64_t r = 0; r < cnt; r += kUnitRows) {
      Unit un;
      un.a_row0 = acc + r;
      un.s_row0 = un.a_row0;
      un.b_row0 = (int64_t)j * b_pad + b_off;
      un.rows = (int32_t)min((int64_t)kUnitRows, cnt - r);
      un.n_items = (int32_t)bp;
      units[nu++] = un;
    }
    acc += ((cnt + kUnitRows - 1) / kUnitRows) * kUnitRows;
  }
  if (t == 1023) {
    a_off[c] = s_rows[1023];
    *n_units = s_units[1023];
    if (rows_out) *rows_out = (int32_t)s_rows[1023];
  }
}

// Stage-1 early-exit bounds per prefix tile (cluster j, tile t): the list's
// ceiling at the tile's first position, scaled and rounded up, clamped at 0
// (ceilings are non-increasing along the list and bound every member's score
// / ||u||, index.py:90-100), and the largest item norm from the tile on.
// (tile_ceil: the same bound for a reordered prefix -- the largest ceiling at
// or after each tile, precomputed by simdex_build_prefix_ordered)
__global__ void prefix_exit_kernel(const double* __restrict__ bounds, int64_t n, int c, int64_t b_pad, int64_t bp,
                                   double si_scale, const float* __restrict__ pnmax, float* __restrict__ exit_c,
                                   float* __restrict__ exit_m, const double* __restrict__ tile_ceil) {
  const int64_t per = b_pad / kTileN;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (int64_t)c * per) return;
  const int64_t j = g / per, pos = (g - j * per) * kTileN;
  const double ceil = tile_ceil ? tile_ceil[g] : (pos < bp ? bounds[j * n + pos] : 0.0);
  exit_c[g] = pos < bp ? fmaxf(0.f, __double2float_ru(ceil * si_scale)) : 0.f;
  float m = 0.f;
  for (int64_t ch = (j * b_pad + pos) >> 5; ch < ((j + 1) * b_pad) >> 5; ++ch) m = fmaxf(m, pnmax[ch]);
  exit_m[g] = m;
}

// packed row r of cluster j: user q_user[q_off[j] + (r - a_off[j])] or padding.
// A warp per 32 packed rows: lane l locates row r0 + l's cluster (binary
// search over a_off) once, then the warp copies the 32 rows' 16-byte vectors
__global__ void ws_rows_kernel(const int64_t* __restrict__ q_user, const int64_t* __restrict__ q_perm,
                               const int64_t* __restrict__ q_off, const int64_t* __restrict__ a_off, int c,
                               int64_t rows_max, const uint16_t* __restrict__ ub, int kp,
                               const float* __restrict__ u_cu, uint16_t* __restrict__ a_pk, float* __restrict__ cu,
                               int64_t* __restrict__ row_user, int64_t* __restrict__ row_out,
                               int32_t* __restrict__ row_cluster) {
  const int lane = threadIdx.x & 31;
  const int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32;
  const int64_t lim = rows_max < a_off[c] ? rows_max : a_off[c];
  if (r0 >= lim) return;
  const int64_t r = r0 + lane;
  int64_t user = -1;
  if (r < lim) {
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
    user = live ? q_user[q_off[j] + i] : -1;
    cu[r] = live ? u_cu[user] : 0.f;
    row_user[r] = user;
    row_out[r] = live ? (q_perm ? q_perm[q_off[j] + i] : q_off[j] + i) : -1;
    row_cluster[r] = j;
  }
  const int vpr = kp / 8;
  for (int e = lane; e < 32 * vpr; e += 32) {
    const int i = e / vpr, v = e - i * vpr;
    const int64_t ui = __shfl_sync(0xffffffffu, user, i);
    if (r0 + i < lim)
      reinterpret_cast<uint4*>(a_pk + (r0 + i) * kp)[v] =
          ui >= 0 ? reinterpret_cast<const uint4*>(ub + ui * kp)[v] : make_uint4(0, 0, 0, 0);
  }
}

// no work sharing (block = 0): every live row goes straight to the full-list
// pass with T0 = -inf (its visited is Algorithm 1's stop position from 0)
__global__ void all_rows_continue_kernel(const int64_t* __restrict__ row_user, int64_t rows, int64_t* __restrict__ cont,
                                         int32_t* __restrict__ cont_n, float* __restrict__ t0) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  t0[r] = -INFINITY;
  const bool live = row_user[r] >= 0;
  const unsigned m = __ballot_sync(__activemask(), live);
  int base = 0;
  const int lane = threadIdx.x & 31, leader = __ffs(__activemask()) - 1;
  if (lane == leader && m) base = atomicAdd(cont_n, __popc(m));
  base = __shfl_sync(__activemask(), base, leader);
  if (live) cont[base + __popc(m & ((1u << lane) - 1u))] = r;
}

// stage 2: pack the continuing rows densely (rows past the count are zero)
// List-order catalogue pass: the continuing rows grouped by cluster.
// Per-cluster counts (one atomic per row), their exclusive scan (one CTA),
// then each continuing row takes a slot in its cluster's 128-padded range.
// (warp-aggregated: the continuing rows arrive in packed order, i.e. mostly
// grouped by cluster, so one atomic per run of equal clusters in a warp)
__global__ void cont_count_kernel(const int64_t* __restrict__ cont, const int32_t* __restrict__ n_cont,
                                  const int32_t* __restrict__ row_cluster, int32_t* __restrict__ cnt) {
  const int64_t nc = *n_cont;
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); b < nc; b += stride) {
    const int64_t i = b + lane;
    const bool v = i < nc;
    const int cl = v ? row_cluster[cont[i]] : -1;
    const unsigned same = __match_any_sync(0xffffffffu, cl);
    if (v && lane == __ffs(same) - 1) atomicAdd(cnt + cl, __popc(same));
  }
}
__global__ void __launch_bounds__(1024) count_scan_kernel(const int32_t* __restrict__ cnt, int c,
                                                          int64_t* __restrict__ off) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int per = (c + 1023) / 1024;
  const int j0 = min(c, t * per), j1 = min(c, j0 + per);
  int64_t v = 0;
  for (int j = j0; j < j1; ++j) v += cnt[j];
  part[t] = v;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t add = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += add;
    __syncthreads();
  }
  int64_t acc = part[t] - v;
  for (int j = j0; j < j1; ++j) {
    off[j] = acc;
    acc += cnt[j];
  }
  if (t == 1023) off[c] = part[1023];
}
// a warp per 4 continuing rows, 8 lanes per row: the row's slot in its
// cluster's range a_off2[cl] + (arrival order), operand row and bookkeeping
__global__ void cont_group_kernel(const int64_t* __restrict__ cont, const int32_t* __restrict__ n_cont,
                                  const int64_t* __restrict__ row_user, const int64_t* __restrict__ row_out,
                                  const int32_t* __restrict__ row_cluster, const float* __restrict__ cu_in,
                                  const float* __restrict__ t0_in, const uint16_t* __restrict__ a_in, int kp,
                                  const int64_t* __restrict__ a_off2, int32_t* __restrict__ cursor,
                                  uint16_t* __restrict__ a2, float* __restrict__ cu2, float* __restrict__ t02,
                                  int64_t* __restrict__ user2, int64_t* __restrict__ out2, int32_t* __restrict__ clus2) {
  // a warp takes 32 continuing rows: slots by one warp-aggregated atomic per
  // run of equal clusters, then the rows are copied 4 at a time (8 lanes each)
  const int lane = threadIdx.x & 31, gl = lane & 7;
  const int64_t nc = *n_cont;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t base = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; base < nc;
       base += nw * 32) {  // warp-uniform trip count (shuffles below)
    const int64_t i = base + lane;
    const bool v = i < nc;
    const int64_t src = v ? cont[i] : 0;
    const int cl = v ? row_cluster[src] : -1;
    const unsigned same = __match_any_sync(0xffffffffu, cl);
    const int leader = __ffs(same) - 1;
    int64_t first = 0;
    if (v && lane == leader) first = a_off2[cl] + atomicAdd(cursor + cl, __popc(same));
    first = __shfl_sync(0xffffffffu, first, leader);
    const int64_t dst = first + __popc(same & ((1u << lane) - 1u));
    if (v) {
      cu2[dst] = cu_in[src];
      t02[dst] = t0_in[src];
      user2[dst] = row_user[src];
      out2[dst] = row_out[src];
      clus2[dst] = cl;
    }
    for (int j = 0; j < 32; j += 4) {
      const int who = j + (lane >> 3);
      const int64_t s_w = __shfl_sync(0xffffffffu, src, who);
      const int64_t d_w = __shfl_sync(0xffffffffu, dst, who);
      if (base + who < nc) {
        const uint4* sr = reinterpret_cast<const uint4*>(a_in + s_w * kp);
        uint4* d = reinterpret_cast<uint4*>(a2 + d_w * kp);
        for (int q = gl; q < kp / 8; q += 8) d[q] = sr[q];
      }
    }
  }
}

__global__ void cont_rows_kernel(const int64_t* __restrict__ cont, const int32_t* __restrict__ n_cont,
                                 int64_t rows_max, const int64_t* __restrict__ row_user,
                                 const int64_t* __restrict__ row_out, const int32_t* __restrict__ row_cluster,
                                 const float* __restrict__ cu_in, const float* __restrict__ t0_in,
                                 const uint16_t* __restrict__ a_in, int kp, uint16_t* __restrict__ a2,
                                 float* __restrict__ cu2, float* __restrict__ t02, int64_t* __restrict__ user2,
                                 int64_t* __restrict__ out2, int32_t* __restrict__ clus2) {
  // 8 lanes per row (a 64-factor fp16 row is 8 x 16 bytes), 4 rows per warp
  const int gl = threadIdx.x & 7;
  const int64_t nc = *n_cont;
  const int64_t lim = min(rows_max, ((nc + kUnitRows - 1) / kUnitRows) * kUnitRows);
  for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3); r < lim;
       r += (int64_t)gridDim.x * (blockDim.x >> 3)) {
  const bool live = r < nc;
  const int64_t src_row = live ? cont[r] : 0;
  const uint4* s = reinterpret_cast<const uint4*>(a_in + src_row * kp);
  uint4* d = reinterpret_cast<uint4*>(a2 + r * kp);
  for (int v = gl; v < kp / 8; v += 8) d[v] = live ? s[v] : make_uint4(0, 0, 0, 0);
  if (gl == 0) {
    cu2[r] = live ? cu_in[src_row] : 0.f;
    t02[r] = live ? t0_in[src_row] : -INFINITY;
    user2[r] = live ? row_user[src_row] : -1;
    out2[r] = live ? row_out[src_row] : -1;
    clus2[r] = live ? row_cluster[src_row] : 0;
  }
  }
}

// Units of `nr` packed rows (count on the device or the host) over the whole
// catalogue.  With seg_out given and fewer row blocks than half the CTA
// slots, the catalogue is cut into S contiguous segments (>= kMinSegTiles
// tiles each) so the units fill the GPU: S brings the unit count to about
// SIMDEX_SPLIT_TARGET units per slot, bounded by the state rows available;
// segment s of row block b keeps its own state rows s * (row blocks * 128) +
// b * 128 + l (segment 0 = the row itself), merged by merge_segments_kernel.
// A segment starts from the rows' initial thresholds, not from what the
// earlier segments reached, so splitting costs work and only pays when the
// unsplit units would leave most CTAs idle (measured: N = 4, 8 shards).
constexpr int kMinSegTiles = 8;
__global__ void units_from_count_kernel(const int32_t* __restrict__ n_rows_dev, int64_t n_rows_host, int64_t ni,
                                        Unit* __restrict__ units, int32_t* __restrict__ n_units, int64_t units_max,
                                        int32_t* __restrict__ seg_out = nullptr, int64_t slots = 0,
                                        int64_t state_rows = 0) {
  const int64_t nr = n_rows_dev ? (int64_t)*n_rows_dev : n_rows_host;
  const int64_t nblk = (nr + kUnitRows - 1) / kUnitRows;
  const int64_t tiles = (ni + kTileN - 1) / kTileN;
  int64_t S = 1;
  if (seg_out && nblk > 0 && 2 * nblk < slots) {  // fewer row blocks than half the CTA slots
    S = (int64_t)SIMDEX_SPLIT_TARGET * slots / nblk;
    S = min(S, tiles / kMinSegTiles);
    S = min(S, state_rows / (nblk * kUnitRows));
    S = min(S, units_max / nblk);
    S = max(S, (int64_t)1);
  }
  const int64_t seg_tiles = (tiles + S - 1) / S;
  S = (tiles + seg_tiles - 1) / seg_tiles;  // every segment non-empty
  const int64_t nunits = nblk * S;
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u == 0) {
    *n_units = (int32_t)nunits;
    if (seg_out) {
      seg_out[0] = (int32_t)S;
      seg_out[1] = (int32_t)seg_tiles;
    }
  }
  if (u >= nunits || u >= units_max) return;
  const int64_t b = u / S, sg = u - b * S;
  Unit un;
  un.a_row0 = b * kUnitRows;
  un.s_row0 = sg * nblk * kUnitRows + b * kUnitRows;
  un.b_row0 = sg * seg_tiles * kTileN;
  un.rows = (int32_t)min((int64_t)kUnitRows, nr - b * kUnitRows);
  un.n_items = (int32_t)min(seg_tiles * kTileN, ni - un.b_row0);
  units[u] = un;
}

// Drop the catalogue segments no row of a block can take anything from (the
// norm-sorted catalogue's early-exit bound of EXM = 1 evaluated at the
// segment's first item against the rows' starting thresholds); their state
// rows are set empty for the merge.  One warp per unit; kept units are
// compacted into `out` (order free).
__global__ void prune_units_kernel(const Unit* __restrict__ in, const int32_t* __restrict__ n_in,
                                   Unit* __restrict__ out, int32_t* __restrict__ n_out, const float* __restrict__ cu,
                                   const float* __restrict__ T0, const float* __restrict__ nmax32, float g_mul,
                                   float e_abs, int32_t* __restrict__ cnt, int32_t* __restrict__ flags,
                                   float* __restrict__ rowT) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  const int64_t n = *n_in;
  for (int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); u < n; u += nw) {
    const Unit un = in[u];
    bool need = un.b_row0 == 0;
    if (!need) {
      const float nm = nmax32[un.b_row0 >> 5];
      for (int l = lane; l < un.rows; l += 32) {
        const float gu = cu[un.a_row0 + l] * g_mul;
        const float bound = fmaf(gu, nm, 2.f * e_abs) * (1.f + 0x1p-20f);
        if (!(bound < T0[un.a_row0 + l])) need = true;
      }
    }
    need = __any_sync(0xffffffffu, need);
    if (need) {
      if (lane == 0) out[atomicAdd(n_out, 1)] = un;
    } else {
      for (int l = lane; l < un.rows; l += 32) {
        cnt[un.s_row0 + l] = 0;
        flags[un.s_row0 + l] = 0;
        rowT[un.s_row0 + l] = -INFINITY;
      }
    }
  }
}

// Segment merge (split row blocks): for every row, the threshold is the
// largest of its segments' (each a valid lower bound of the K-th score), the
// segments' candidates reaching it are appended to segment 0's buffer (the
// row's own) with their positions made absolute (a unit stores positions
// relative to its first item row), a row whose candidates do not fit is
// flagged (exact fallback).
__global__ void merge_segments_kernel(const int32_t* __restrict__ n_rows_dev, const int32_t* __restrict__ seg,
                                      int cap, int32_t* __restrict__ cid, float* __restrict__ chi,
                                      int32_t* __restrict__ cnt, int32_t* __restrict__ flags, float* __restrict__ rowT) {
  // a warp per row, a lane per segment (a thread per row walked S x count
  // dependent loads: 0.13 ms for the optimizer's 1,200-row sample)
  const int S = seg[0];
  if (S <= 1) return;
  const int32_t seg_items = seg[1] * kTileN;
  const int64_t nr = *n_rows_dev;
  const int64_t stride = ((nr + kUnitRows - 1) / kUnitRows) * kUnitRows;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < nr; r += nwarps) {
    float T = -INFINITY;
    int fl = 0;
    for (int s = lane; s < S; s += 32) {
      T = fmaxf(T, rowT[r + s * stride]);
      fl |= flags[r + s * stride];
    }
    for (int o = 16; o > 0; o >>= 1) T = fmaxf(T, __shfl_xor_sync(0xffffffffu, T, o));
    fl = __any_sync(0xffffffffu, fl != 0) ? 1 : 0;
    int c = cnt[r];
    for (int s0 = 1; s0 < S && !fl; s0 += 32) {
      const int s = s0 + lane;
      const int64_t q = r + (int64_t)s * stride;
      const int cq = s < S ? cnt[q] : 0;
      const int cmax = __reduce_max_sync(0xffffffffu, cq);
      for (int e = 0; e < cmax; ++e) {  // appended in (entry, segment) order: deterministic
        float h = 0.f;
        bool keep = false;
        if (e < cq) {
          h = chi[q * cap + e];
          keep = h >= T;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (!bal) continue;
        if (c + __popc(bal) > cap) {
          fl = 1;
          break;
        }
        if (keep) {
          const int pos = c + __popc(bal & ((1u << lane) - 1u));
          chi[r * cap + pos] = h;
          cid[r * cap + pos] = cid[q * cap + e] + s * seg_items;
        }
        c += __popc(bal);
      }
    }
    __syncwarp();
    if (lane == 0) {
      cnt[r] = c;
      flags[r] = fl;
      rowT[r] = T;
    }
  }
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// A tensor map is a pure function of (address, rows, kp): cached per thread,
// so a serving call encodes nothing after its first run.
struct MapKey {
  const void* ptr;
  int64_t rows;
  int kp;
  bool operator<(const MapKey& o) const {
    return ptr != o.ptr ? ptr < o.ptr : rows != o.rows ? rows < o.rows : kp < o.kp;
  }
};

int encode_map(CUtensorMap* m, const void* ptr, int64_t rows, int kp);

int make_map(CUtensorMap* m, const void* ptr, int64_t rows, int kp) {
  static thread_local std::map<MapKey, CUtensorMap> cache;
  const MapKey key{ptr, rows, kp};
  auto it = cache.find(key);
  if (it != cache.end()) {
    *m = it->second;
    return SIMDEX_OK;
  }
  const int rc = encode_map(m, ptr, rows, kp);
  if (rc) return rc;
  if (cache.size() >= 512) cache.clear();
  cache[key] = *m;
  return SIMDEX_OK;
}

int encode_map(CUtensorMap* m, const void* ptr, int64_t rows, int kp) {
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
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d) rows=%lld kp=%d", (int)r, (long long)rows, kp);
    return SIMDEX_ECUDA;
  }
  return SIMDEX_OK;
}

double eps_for(int kp) {
  return std::ldexp(1.0, -10) + std::ldexp(1.0, -22) + (kp + 16) * std::ldexp(1.0, -22) + std::ldexp(1.0, -20);
}

int kt_for(int k_eff) {
  if (k_eff <= 1) return 1;
  if (k_eff <= 2) return 2;
  if (k_eff <= 4) return 4;
  if (k_eff == 5) return 5;  // exact sizes for the BASELINE depths K = 5, 10
  if (k_eff <= 8) return 8;
  if (k_eff == 10) return 10;
  if (k_eff <= 16) return 16;
  if (k_eff <= 32) return 32;
  if (k_eff == 50) return 50;  // BASELINE depth K = 50
  if (k_eff <= 64) return 64;
  return 0;
}

int cap_for(int k_eff) {
  const int kt = kt_for(k_eff);
  if (kt > 0) return kt <= 32 ? 128 : 256;  // T exact-current: the band + 32 free slots
  int c = 4 * k_eff + 64;
  int p = 64;
  while (p < c) p <<= 1;
  return p > kMaxCap ? kMaxCap : p;
}

struct GemmGeometry {
  int kb, stages;
  size_t smem;
  int ctas_per_sm;  // kCtasPerSm, or 1 when a CTA's operands need more than half the SM's shared memory
};

int geometry(int kp, GemmGeometry* g) {
  g->kb = kp / 64;
  const size_t fixed = 1024 + kMTiles * (size_t)g->kb * kSlab + 512;
  g->ctas_per_sm = kCtasPerSm;
  size_t budget = kCtasPerSm == 1 ? 225 * 1024 : 112 * 1024;
  if (fixed + 2 * (size_t)g->kb * kSlab > budget) {  // fewer than 2 stages would fit: one CTA per SM
    g->ctas_per_sm = 1;
    budget = 225 * 1024;
  }
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

template <int KT>
int launch_gemm_kt(const CUtensorMap& ma, const CUtensorMap& mb, const TopkParams& p, const GemmGeometry& g, int grid,
                   const char* prof, cudaStream_t s) {
  auto kern = p.exit_c ? gemm_topk_kernel<KT, 2> : p.norm_sorted ? gemm_topk_kernel<KT, 1> : gemm_topk_kernel<KT, 0>;
  static size_t set_for[16][3] = {};  // per device and exit mode: largest shared-memory size already allowed
  const int em = p.exit_c ? 2 : p.norm_sorted ? 1 : 0;
  int dev = 0;
  cudaGetDevice(&dev);
  size_t& done = set_for[dev & 15][em];
  if (g.smem > done) {
    SIMDEX_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem));
    done = g.smem;
  }
  ProfileScope _prof(prof, s);
  kern<<<grid, kThreads, g.smem, s>>>(ma, mb, p);
  _prof.end();
  SIMDEX_LAUNCH_CHECK("gemm_topk");
  return SIMDEX_OK;
}

// prof: the simdex_profile name of this launch (gemm_topk, gemm_topk_prefix,
// gemm_topk_full, gemm_assign)
int launch_gemm(const CUtensorMap& ma, const CUtensorMap& mb, const TopkParams& p, const GemmGeometry& g, int grid,
                const char* prof, cudaStream_t s) {
  if (p.debug_out) return launch_gemm_kt<-1>(ma, mb, p, g, grid, prof, s);
  switch (kt_for(p.k_eff)) {
    case 1: return launch_gemm_kt<1>(ma, mb, p, g, grid, prof, s);
    case 2: return launch_gemm_kt<2>(ma, mb, p, g, grid, prof, s);
    case 4: return launch_gemm_kt<4>(ma, mb, p, g, grid, prof, s);
    case 5: return launch_gemm_kt<5>(ma, mb, p, g, grid, prof, s);
    case 8: return launch_gemm_kt<8>(ma, mb, p, g, grid, prof, s);
    case 10: return launch_gemm_kt<10>(ma, mb, p, g, grid, prof, s);
    case 16: return launch_gemm_kt<16>(ma, mb, p, g, grid, prof, s);
    case 32: return launch_gemm_kt<32>(ma, mb, p, g, grid, prof, s);
    case 50: return launch_gemm_kt<50>(ma, mb, p, g, grid, prof, s);
    case 64: return launch_gemm_kt<64>(ma, mb, p, g, grid, prof, s);
    default: return launch_gemm_kt<0>(ma, mb, p, g, grid, prof, s);
  }
}

template <int LPR>
int launch_finalize_lpr(const FinalizeParams& fp, int64_t rows, const char* prof, cudaStream_t s) {
  constexpr int RPW = 32 / LPR;
  const size_t per_row = ((size_t)fp.pow2 * 12 + (size_t)fp.f * 8 + 15) & ~size_t(15);
  int warps = 8;
  while (warps > 1 && per_row * RPW * warps > 100 * 1024) warps >>= 1;
  const size_t smem = per_row * RPW * warps;
  if (smem > 200 * 1024) {
    set_error("finalize: candidate buffer too large");
    return SIMDEX_EUNSUPPORTED;
  }
  static size_t set_for[16] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (smem > set_for[dev & 15]) {
    SIMDEX_CUDA(cudaFuncSetAttribute(finalize_kernel<LPR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    set_for[dev & 15] = smem;
  }
  ProfileScope _prof(prof, s);
  finalize_kernel<LPR><<<(unsigned)ceil_div(rows, RPW * warps), 32 * warps, smem, s>>>(fp);
  _prof.end();
  SIMDEX_LAUNCH_CHECK("finalize");
  return SIMDEX_OK;
}

int launch_finalize(const FinalizeParams& fp, int64_t rows, const char* prof, cudaStream_t s) {
  return fp.k_eff > 32 ? launch_finalize_lpr<32>(fp, rows, prof, s) : launch_finalize_lpr<8>(fp, rows, prof, s);
}

// Candidate buffers + per-row state for up to `rows` packed rows (carved
// out of the context workspace).
struct RowState {
  int32_t *cid = nullptr, *cnt = nullptr, *flags = nullptr;
  float *lo = nullptr, *hi = nullptr, *rowT = nullptr;
  int cap = 0;
  void add(Workspace& ws, int64_t rows, int k_eff) {
    cap = cap_for(k_eff);
    ws.add(&cid, (size_t)rows * cap);
    ws.add(&hi, (size_t)rows * cap);
    ws.add(&lo, kt_for(k_eff) > 0 ? 1 : (size_t)rows * cap);
    ws.add(&cnt, rows);
    ws.add(&flags, rows);
    ws.add(&rowT, rows);
  }
};

TopkParams make_params(const RowState& st, const Unit* units, const int32_t* n_units, const float* inrm,
                       const float* inmax, const float* cu, const GemmGeometry& g, int f, int k_eff) {
  TopkParams p{};
  p.units = units;
  p.n_units = n_units;
  p.item_nrm = inrm;
  p.item_nmax32 = inmax;
  p.row_cu = cu;
  p.e_abs = (float)(std::ldexp((double)(((f + 63) / 64) * 64), -22) + std::ldexp((double)(f + 1), -124));
  p.kb = g.kb;
  p.k_steps = (f + 15) / 16;
  p.stages = g.stages;
  p.cap = st.cap;
  p.k_eff = k_eff;
  p.cand_id = st.cid;
  p.cand_lo = st.lo;
  p.cand_hi = st.hi;
  p.row_count = st.cnt;
  p.row_flags = st.flags;
  p.row_T_out = st.rowT;
  p.g_mul = (float)((1.0 / eps_for(((f + 63) / 64) * 64) + 2.0) * (1.0 + 0x1p-20));
  p.u_mul = (float)((1.0 / eps_for(((f + 63) / 64) * 64)) * (1.0 + 0x1p-20));

  return p;
}

// Cooperative rescoring (finalize_kernel): on whenever the kernel's
// conditions hold (8 lanes per row, exact float32 copies, even f in [36, 64]).
// Measured against a lane per candidate: cfg2 prefix finalize 0.338 -> 0.291
// ms at K = 10, 0.232 -> 0.205 at K = 5, 0.173 -> 0.152 at K = 1; cfg4 1.19
// -> 1.09 at K = 10, 0.66 -> 0.58 at K = 1.  SIMDEX_FIN_COOP_FORCE=0/1: A/B.
int finalize_coop(int64_t, int, int) {
  if (const char* e = getenv("SIMDEX_FIN_COOP_FORCE")) return atoi(e);
  return 1;
}

int pow2_at_least(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}

// fallback_visited launches grid-stride: the overflow count lives on the
// device, a fixed grid covers any count
constexpr int kFallbackGrid = 64;

}  // namespace

// Work-sharing call statistics (simdex_ws_stats): queries, rows that went on
// past B, prefix length, list length, factors -- enough for the caller to
// count the algorithmic tensor work of the last call.  The continuing-row
// count reaches a pinned host slot of the context asynchronously; it is
// valid once the stream has synchronised.
static thread_local int64_t g_ws_stats[5] = {0, 0, 0, 0, 0};
static thread_local const int64_t* g_ws_cont_slot = nullptr;
void record_ws_stats(int64_t nq, const int64_t* n_cont_slot, int64_t n_cont, int64_t bp, int64_t n, int64_t f) {
  g_ws_stats[0] = nq;
  g_ws_stats[1] = n_cont;
  g_ws_stats[2] = bp;
  g_ws_stats[3] = n;
  g_ws_stats[4] = f;
  g_ws_cont_slot = n_cont_slot;
}
void read_ws_stats(int64_t* out) {
  for (int i = 0; i < 5; ++i) out[i] = g_ws_stats[i];
  if (g_ws_cont_slot) out[1] = *g_ws_cont_slot;
}

// rows of this thread's last serving call that took the exact float64
// fallback (band wider than the candidate buffer); pinned host slot 1 of the
// context, valid once the stream has synchronised
static thread_local const int64_t* g_fallback_slot = nullptr;
int record_fallback_count(Ctx* ctx, const int32_t* over_n, cudaStream_t s) {
  int64_t* host = ctx_host_slots(ctx);
  g_fallback_slot = &host[1];
  SIMDEX_CUDA(cudaMemcpyAsync(&host[1], over_n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  return SIMDEX_OK;
}
int64_t read_fallback_count() { return g_fallback_slot ? *g_fallback_slot : 0; }

// (user, item) pairs the tensor-core launches of this thread's last serving
// call actually multiplied (early exits skip tiles): [first launch, second
// launch] -- pinned host slots 2, 3 of the context, valid after synchronisation
static thread_local const int64_t* g_pairs_slot = nullptr;
int record_pairs(Ctx* ctx, const unsigned long long* dev2, cudaStream_t s) {
  int64_t* host = ctx_host_slots(ctx);
  g_pairs_slot = &host[2];
  SIMDEX_CUDA(cudaMemcpyAsync(&host[2], dev2, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  return SIMDEX_OK;
}
// the four statistic slots of a work-sharing call in ONE copy: a device block
// laid out as the host slots [continuing rows, overflow rows, pairs 1, pairs 2]
// (the counts int32 in the low halves of zeroed int64 slots)
int record_stat_block(Ctx* ctx, const int64_t* blk, cudaStream_t s) {
  int64_t* host = ctx_host_slots(ctx);
  g_fallback_slot = &host[1];
  g_pairs_slot = &host[2];
  SIMDEX_CUDA(cudaMemcpyAsync(host, blk, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  return SIMDEX_OK;
}
void read_pairs(int64_t* out2) {
  out2[0] = g_pairs_slot ? g_pairs_slot[0] : 0;
  out2[1] = g_pairs_slot ? g_pairs_slot[1] : 0;
}

// Brute-force fused path (topk_matmul).  No allocation, no host round trip
// (options & SIMDEX_MM_NORM_AUTO excepted: it reads two norms to decide the
// early exit).
int gemm_topk_brute(const double* users, const float* users32, const uint16_t* ub, const double* u_norm, int64_t nu, const double* items,
                    const float* items32, const uint16_t* ib, const double* i_norm, const int32_t* item_perm, int64_t ib_rows, int64_t ni,
                    int32_t f, int32_t kp, int32_t su, const int32_t* u_exp, int32_t si, int32_t k, int32_t* out_ids,
                    double* out_scores, int64_t* heap_ops, float* debug_out, int32_t options, Ctx* ctx,
                    cudaStream_t s) {
  const int k_eff = (int)(k < ni ? k : ni);
  GemmGeometry g;
  int rc = geometry(kp, &g);
  if (rc) return rc;
  const int64_t nu_pad = ceil_div(nu, 256) * 256;
  const int64_t ni_pad = ib_rows > 0 ? ib_rows : ceil_div(ni, 256) * 256;  // rows of the item operand
  const int64_t nunits = ceil_div(nu, kUnitRows);
  const bool fallback = debug_out == nullptr;
  Workspace ws(ctx, s);
  RowState st;
  st.add(ws, nu_pad, k_eff);
  Unit* units;
  int32_t *n_units, *over_n;
  float *cu, *inrm, *inmax;
  int64_t *over_list, *over_out;
  double* slab = nullptr;
  ws.add(&units, nunits);
  ws.add(&n_units, 1);
  ws.add(&cu, nu_pad);
  ws.add(&inrm, ni_pad);
  ws.add(&inmax, ni_pad / 32);
  ws.add(&over_n, 1);
  ws.add(&over_list, nu);
  ws.add(&over_out, nu);
  if (fallback) ws.add(&slab, (size_t)exact_slab_ctas(ni) * ni);
  unsigned long long* pairs;
  ws.add(&pairs, 2);
  if ((rc = ws.commit())) return rc;
  SIMDEX_CUDA(cudaMemsetAsync(pairs, 0, 2 * sizeof(unsigned long long), s));
  const double eps = eps_for(kp);
  units_from_count_kernel<<<(unsigned)ceil_div(nunits, 256), 256, 0, s>>>(nullptr, nu, ni, units, n_units,
                                                                          nunits);
  SIMDEX_LAUNCH_CHECK("units");
  row_cu_kernel<<<(unsigned)ceil_div(nu_pad, 256), 256, 0, s>>>(u_norm, nu, nu_pad, eps * std::ldexp(1.0, su), cu,
                                                                nullptr, u_exp);
  SIMDEX_LAUNCH_CHECK("row_cu");
  item_nrm_kernel<<<(unsigned)ceil_div(ni_pad / 32, 8), 256, 0, s>>>(i_norm, ni, ni_pad, std::ldexp(1.0, si), inrm,
                                                                      inmax);
  SIMDEX_LAUNCH_CHECK("item_nrm");
  CUtensorMap ma, mb;
  if ((rc = make_map(&ma, ub, nu_pad, kp))) return rc;
  if ((rc = make_map(&mb, ib, ni_pad, kp))) return rc;
  TopkParams p = make_params(st, units, n_units, inrm, inmax, cu, g, f, k_eff);
  p.heap_ops = heap_ops;
  p.debug_out = debug_out;
  p.debug_ld = ni;
  p.pairs_out = pairs;
  // early exit pays when the catalogue's norms are skewed (the streaming
  // kernel with exit checks is slower when no tile can be skipped): the
  // caller decides once per operand (SIMDEX_MM_NORM_EXIT); NORM_AUTO reads
  // the norm-sorted operand's largest and median norms here
  p.norm_sorted = 0;
  if (item_perm != nullptr && !debug_out && ni >= 2 * kTileN && !getenv("SIMDEX_NO_EARLY_EXIT")) {
    if (options & SIMDEX_MM_NORM_EXIT) {
      p.norm_sorted = 1;
    } else if (options & SIMDEX_MM_NORM_AUTO) {
      double nn[2];
      SIMDEX_CUDA(cudaMemcpyAsync(&nn[0], i_norm, sizeof(double), cudaMemcpyDeviceToHost, s));
      SIMDEX_CUDA(cudaMemcpyAsync(&nn[1], i_norm + ni / 2, sizeof(double), cudaMemcpyDeviceToHost, s));
      SIMDEX_CUDA(cudaStreamSynchronize(s));
      p.norm_sorted = nn[1] < 0.6 * nn[0];
    }
  }
  const int grid = (int)(nunits < g.ctas_per_sm * sm_count() ? nunits : g.ctas_per_sm * sm_count());
  if ((rc = launch_gemm(ma, mb, p, g, grid, "gemm_topk", s))) return rc;
  if (debug_out) return SIMDEX_OK;
  SIMDEX_CUDA(cudaMemsetAsync(over_n, 0, sizeof(int32_t), s));
  FinalizeParams fp{};
  fp.mode = kBrute;
  fp.total_rows = nu;
  fp.nu = nu;
  fp.users = users;
  fp.users32 = users32;
  fp.items = items;
  fp.items32 = items32;
  fp.f = f;
  fp.n = ni;
  fp.k_eff = k_eff;
  fp.cap = st.cap;
  fp.cand_id = st.cid;
  fp.cand_hi = st.hi;
  fp.row_T = st.rowT;
  fp.row_count = st.cnt;
  fp.row_flags = st.flags;
  fp.out_ids = out_ids;
  fp.out_scores = out_scores;
  fp.over_list = over_list;
  fp.over_out = over_out;
  fp.over_n = over_n;
  fp.item_perm = item_perm;
  fp.pow2 = pow2_at_least(std::min(st.cap, std::max(64, 2 * k_eff + 32)));
  fp.coop = finalize_coop(ni, f, k_eff);
  if ((rc = launch_finalize(fp, nu, "finalize", s))) return rc;
  if ((rc = record_fallback_count(ctx, over_n, s))) return rc;
  if ((rc = record_pairs(ctx, pairs, s))) return rc;
  // band overflow (rare): exact float64 rows, the count read on the device
  return exact_topk_devcount(users, users32, items, items32, ni, f, over_list, nullptr, over_n, k, over_out,
                             out_ids, out_scores, slab, s);
}

// Work-sharing path (query_batch, work_sharing=True):
//   stage 1  every cluster's first B' list items x that cluster's queried
//            users (segmented tensor-core product, certified top-K); users
//            whose K-th beats the ceiling at B' are done (visited = B');
//   stage 2  the remaining users x the whole catalogue (certified top-K), and
//            visited from the closed form of Algorithm 1's stop position.
// Every buffer comes from the context workspace and every count stays on the
// device: the call enqueues its kernels and returns (CUDA-graph capturable).
int gemm_topk_ws(const double* users, const float* users32, const uint16_t* ub, const double* unorm, int64_t nu, const double* items,
                 const float* items32, const uint16_t* ib, const double* i_norm, const int32_t* item_perm, int64_t ib_rows, int64_t ni,
                 int32_t f, int32_t kp, int32_t su, const int32_t* u_exp, int32_t si,
                 const int32_t* list_ids, const int32_t* list_pos, const double* bounds, int32_t c, int64_t block,
                 const uint16_t* prefix_b, const double* prefix_norm, const int32_t* prefix_ids,
                 const double* prefix_tile_ceil, int64_t b_pad, const int64_t* q_user,
                 const int64_t* q_perm, const int64_t* q_off, int64_t nq, int32_t k, int32_t* out_ids,
                 double* out_scores, int64_t* out_visited, int32_t options, Ctx* ctx, cudaStream_t s) {
  const int k_eff = (int)(k < ni ? k : ni);
  const bool no_ws = block == 0;  // every query walks the whole list (query_batch(work_sharing=False))
  const int64_t bp = block < ni ? block : ni;
  if (no_ws) b_pad = 0;
  GemmGeometry g;
  int rc = geometry(kp, &g);
  if (rc) return rc;
  const int64_t rows_max = nq + (int64_t)c * kUnitRows;
  const int64_t units_max = ceil_div(nq, kUnitRows) + c;
  const int64_t ni_pad = ib_rows > 0 ? ib_rows : ceil_div(ni, 256) * 256;
  const double eps = eps_for(kp);
  const bool stats = getenv("SIMDEX_STATS") != nullptr;
  const bool prefix_exit = !no_ws && (options & SIMDEX_WS_PREFIX_EXIT) && !getenv("SIMDEX_NO_EARLY_EXIT");
  const bool stage2 = no_ws || bp < ni;
  const int64_t rows2 = ceil_div(nq, kUnitRows) * kUnitRows;  // bound on the continuing rows
  const int64_t units2 = rows2 / kUnitRows;
  const int64_t nt = (int64_t)c * (b_pad / kTileN);

  const CtxSetup held_before = *ctx_setup(ctx);  // what the previous call on this context left
  // per-cluster full lists handed to this call (simdex_ctx_set_full_lists): the
  // continuing users scan their own cluster's list from B' in list order
  const uint16_t* full_b = held_before.full_b;
  const double* full_norm = held_before.full_norm;
  const int64_t bf_pad = held_before.bf_pad;
  ctx_setup(ctx)->full_b = nullptr;
  ctx_setup(ctx)->full_norm = nullptr;
  ctx_setup(ctx)->bf_pad = 0;
  // (from K = 8 on and for large query sets: at K = 1, 5 the continuing users
  // are few and the grouping and per-cluster units cost more than the shorter
  // scan saves; for a multi-GPU share of ~30k users a few per-cluster units
  // running to their longest walk set the time, where the norm-sorted pass
  // cuts the catalogue into segments -- measured)
  const bool list2 = SIMDEX_LIST_STAGE2 && stage2 && !no_ws && full_b && full_norm && bf_pad >= ni && bp % kTileN == 0 &&
                     k_eff >= SIMDEX_LIST_MIN_K && nq >= SIMDEX_LIST_MIN_Q && !getenv("SIMDEX_NO_LIST_STAGE2") &&
                     !getenv("SIMDEX_STATS");
  const int64_t rows_s2 = list2 ? rows_max : rows2;  // stage-2 packed rows (cluster-padded in list mode)
  Workspace ws(ctx, s);
  RowState st;
  st.add(ws, rows_max, k_eff);
  Unit* units;
  int32_t *n_units, *cont_n, *over_n, *rclus, *clus2 = nullptr;
  float *cu, *ucu, *pnrm = nullptr, *pnmax = nullptr, *inrm = nullptr, *inmax = nullptr, *cu2 = nullptr, *t0,
        *t02 = nullptr, *exit_c = nullptr, *exit_m = nullptr;
  int64_t *a_off, *row_user, *row_out, *cont, *over_list, *over_out, *user2 = nullptr, *out2 = nullptr;
  uint16_t *a_pk, *a2 = nullptr;
  double* slab = nullptr;
  ws.add(&units, units_max > units2 ? units_max : units2);
  ws.add(&n_units, 1);
  int32_t *seg_n, *n_units_raw, *n_units_s2;
  Unit *units_raw, *units_s2;  // stage 2's own unit lists (stage 1's are kept for a reused setup)
  ws.add(&units_s2, units_max > units2 ? units_max : units2);
  ws.add(&n_units_s2, 1);
  ws.add(&seg_n, 2);
  ws.add(&n_units_raw, 1);
  ws.add(&units_raw, units_max > units2 ? units_max : units2);
  ws.add(&a_off, c + 1);
  ws.add(&a_pk, (size_t)rows_max * kp);
  ws.add(&cu, rows_max);
  ws.add(&ucu, nu);
  ws.add(&row_user, rows_max);
  ws.add(&row_out, rows_max);
  ws.add(&rclus, rows_max);
  ws.add(&cont, rows_max);
  ws.add(&t0, rows_max);
  int64_t* statblk;  // [cont_n, over_n, pairs[2]] as host slots (record_stat_block)
  ws.add(&statblk, 4);
  ws.add(&over_list, rows_max);
  ws.add(&over_out, rows_max);
  if (!no_ws) {
    ws.add(&pnrm, (size_t)c * b_pad + 1);
    ws.add(&pnmax, (size_t)c * b_pad / 32 + 1);
  }
  if (prefix_exit) {
    ws.add(&exit_c, nt);
    ws.add(&exit_m, nt);
  }
  int64_t *q_off2 = nullptr, *a_off2 = nullptr, *over1_list = nullptr, *over1_out = nullptr;
  int32_t *cnt2 = nullptr, *cur2 = nullptr, *rows2_n = nullptr, *over1_n = nullptr;
  float *fnrm = nullptr, *fnmax = nullptr, *exit_c2 = nullptr, *exit_m2 = nullptr;
  const int64_t nt2 = list2 ? (int64_t)c * (bf_pad / kTileN) : 0;
  if (list2) {
    ws.add(&q_off2, c + 1);
    ws.add(&a_off2, c + 1);
    ws.add(&cnt2, c);
    ws.add(&cur2, c);
    ws.add(&rows2_n, 4);  // [0] grouped rows, [1] prefix-overflow rows
    ws.add(&over1_list, rows_max);
    ws.add(&over1_out, rows_max);
    ws.add(&fnrm, (size_t)c * bf_pad);
    ws.add(&fnmax, (size_t)c * bf_pad / 32);
    ws.add(&exit_c2, nt2);
    ws.add(&exit_m2, nt2);
  }
  if (stage2) {
    ws.add(&a2, (size_t)rows_s2 * kp);
    ws.add(&cu2, rows_s2);
    ws.add(&t02, rows_s2);
    ws.add(&user2, rows_s2);
    ws.add(&out2, rows_s2);
    ws.add(&clus2, rows_s2);
    ws.add(&inrm, ni_pad);
    ws.add(&inmax, ni_pad / 32);
    ws.add(&slab, (size_t)exact_slab_ctas(ni) * ni);
  }
  if ((rc = ws.commit())) return rc;
  int64_t* host = ctx_host_slots(ctx);
  cont_n = reinterpret_cast<int32_t*>(statblk);
  over_n = reinterpret_cast<int32_t*>(statblk + 1);
  unsigned long long* pairs = reinterpret_cast<unsigned long long*>(statblk + 2);
  SIMDEX_CUDA(cudaMemsetAsync(statblk, 0, 4 * sizeof(int64_t), s));

  // per-query-set setup (units, packed rows and their bands, prefix norms):
  // skipped when the context holds it for this query set (its token), these
  // inputs and this arena (simdex_ctx_set_query_token)
  CtxSetup* cs = ctx_setup(ctx);
  const int64_t qtok = cs->query_token;
  cs->query_token = 0;  // consumed by this call
  uint64_t sig = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { sig = (sig ^ v) * 1099511628211ull; };
  for (const void* ptrv : {(const void*)q_user, (const void*)q_perm, (const void*)q_off, (const void*)ub,
                           (const void*)unorm, (const void*)u_exp, (const void*)prefix_norm, (const void*)i_norm,
                           (const void*)full_b, (const void*)full_norm})
    mix((uint64_t)(uintptr_t)ptrv);
  for (int64_t v : {nq, nu, (int64_t)c, b_pad, bp, (int64_t)kp, (int64_t)su, (int64_t)si, rows_max, ni, ni_pad,
                    (int64_t)k_eff, (int64_t)no_ws, bf_pad, (int64_t)list2})
    mix((uint64_t)v);
  // (the held setup is what the previous call on this context left: commit()
  // cleared it, so compare against the value saved before the commit)
  const bool reuse = qtok != 0 && held_before.held_token == qtok && held_before.held_gen == ctx_arena_gen(ctx) &&
                     held_before.held_sig == sig && !getenv("SIMDEX_NO_SETUP_REUSE");
  if (!reuse) {
    ws_units_kernel<<<1, 1024, 0, s>>>(q_off, c, b_pad, bp, a_off, units, n_units);
    SIMDEX_LAUNCH_CHECK("ws_units");
    row_cu_kernel<<<(unsigned)ceil_div(nu, 256), 256, 0, s>>>(unorm, nu, nu, eps * std::ldexp(1.0, su), ucu,
                                                              nullptr, u_exp);
    SIMDEX_LAUNCH_CHECK("row_cu");
    // rows past a_off[c] stay "padding" (row_user = -1) and are skipped by finalize
    SIMDEX_CUDA(cudaMemsetAsync(row_user, 0xff, sizeof(int64_t) * rows_max, s));
    ws_rows_kernel<<<(unsigned)ceil_div(rows_max, 256), 256, 0, s>>>(q_user, q_perm, q_off, a_off, c, rows_max, ub,
                                                                     kp, ucu, a_pk, cu, row_user, row_out, rclus);
    SIMDEX_LAUNCH_CHECK("ws_rows");
    if (!no_ws) {
      item_nrm_kernel<<<(unsigned)ceil_div((int64_t)c * b_pad / 32, 8), 256, 0, s>>>(
          prefix_norm, (int64_t)c * b_pad, (int64_t)c * b_pad, std::ldexp(1.0, si), pnrm, pnmax);
      SIMDEX_LAUNCH_CHECK("item_nrm");
    }
    if (list2) {  // the full lists' scaled norms and per-tile stop bounds (list ceilings)
      item_nrm_kernel<<<(unsigned)ceil_div((int64_t)c * bf_pad / 32, 8), 256, 0, s>>>(
          full_norm, (int64_t)c * bf_pad, (int64_t)c * bf_pad, std::ldexp(1.0, si), fnrm, fnmax);
      SIMDEX_LAUNCH_CHECK("item_nrm");
      prefix_exit_kernel<<<(unsigned)ceil_div(nt2, 256), 256, 0, s>>>(bounds, ni, c, bf_pad, ni, std::ldexp(1.0, si),
                                                                      fnmax, exit_c2, exit_m2, nullptr);
      SIMDEX_LAUNCH_CHECK("prefix_exit");
    }
  }
  if (qtok != 0) {  // the arena now holds this query set's setup
    cs->held_token = qtok;
    cs->held_gen = ctx_arena_gen(ctx);
    cs->held_sig = sig;
  }
  int grid = 0;
  if (!no_ws) {
    CUtensorMap ma, mb;
    if ((rc = make_map(&ma, a_pk, rows_max, kp))) return rc;
    if ((rc = make_map(&mb, prefix_b, (int64_t)c * b_pad, kp))) return rc;
    TopkParams p = make_params(st, units, n_units, pnrm, pnmax, cu, g, f, k_eff);
    p.pairs_out = pairs;
    // early exit on the cluster ceilings (Algorithm 1's own stop bound): a
    // unit stops once every row's threshold exceeds ||u|| x the next tile's
    // ceiling; the prefix top-K is unchanged (later items cannot reach it)
    if (prefix_exit) {
      prefix_exit_kernel<<<(unsigned)ceil_div(nt, 256), 256, 0, s>>>(bounds, ni, c, b_pad, bp, std::ldexp(1.0, si),
                                                                     pnmax, exit_c, exit_m, prefix_tile_ceil);
      SIMDEX_LAUNCH_CHECK("prefix_exit");
      p.norm_sorted = 1;
      p.exit_c = exit_c;
      p.exit_m = exit_m;
      p.first_all = prefix_ids == nullptr && !getenv("SIMDEX_FIRST_FILTERED");  // list-order prefix; a hybrid one
                                                                               // keeps the threshold-filtered stores
      // a two-stage ring for the exit kernel: the tiles already in flight when
      // a unit ends are wasted work, and the epilogue (not the loads) sets the
      // pace (prefix pass at cfg4 K=10: 0.55 -> 0.46 ms, K=1: 0.36 -> 0.27 ms
      // against the 5-stage ring)
      if (p.stages > 2) p.stages = 2;
    }
    Scratch<int64_t> hops;
    if (stats) {
      SIMDEX_CUDA(hops.alloc(rows_max, s));
      SIMDEX_CUDA(cudaMemsetAsync(hops.p, 0, sizeof(int64_t) * rows_max, s));
      p.heap_ops = hops.p;
    }
    grid = (int)(units_max < g.ctas_per_sm * sm_count() ? units_max : g.ctas_per_sm * sm_count());
    if ((rc = launch_gemm(ma, mb, p, g, grid, "gemm_topk_prefix", s))) return rc;
    if (stats) {
      std::vector<int64_t> hh(rows_max);
      SIMDEX_CUDA(cudaMemcpy(hh.data(), hops.p, sizeof(int64_t) * rows_max, cudaMemcpyDeviceToHost));
      int64_t tot = 0;
      for (auto v : hh) tot += v;
      fprintf(stderr, "[simdex] stage1 appends per query %.2f\n", (double)tot / (double)nq);
    }
  }

  // (cont_n and over_n were zeroed with the statistics block)
  FinalizeParams fp{};
  fp.mode = kPrefix;
  fp.total_rows = rows_max;
  fp.row_user = row_user;
  fp.row_out = row_out;
  fp.row_cluster = rclus;
  fp.nu = nu;
  fp.users = users;
  fp.users32 = users32;
  fp.items = items;
  fp.items32 = items32;
  fp.f = f;
  fp.list_ids = list_ids;
  fp.list_pos = list_pos;
  fp.bounds = bounds;
  fp.unorm = unorm;
  fp.n = ni;
  fp.prefix = bp;
  fp.k_eff = k_eff;
  fp.cap = st.cap;
  fp.cand_id = st.cid;
  fp.cand_hi = st.hi;
  fp.row_T = st.rowT;
  fp.row_count = st.cnt;
  fp.row_flags = st.flags;
  fp.out_ids = out_ids;
  fp.out_scores = out_scores;
  fp.out_visited = out_visited;
  fp.row_T0_out = t0;
  fp.t0_scale = std::ldexp(1.0, su + si);
  fp.u_exp = u_exp;
  fp.prefix_ids = prefix_ids;
  fp.prefix_ld = b_pad;
  fp.cont_list = cont;
  fp.cont_n = cont_n;
  fp.over_list = over_list;
  fp.over_out = over_out;
  fp.over_n = over_n;
  fp.pow2 = pow2_at_least(std::min(st.cap, std::max(64, 2 * k_eff + 32)));
  fp.coop = finalize_coop(ni, f, k_eff);
  if (list2) {
    SIMDEX_CUDA(cudaMemsetAsync(rows2_n, 0, 4 * sizeof(int32_t), s));
    over1_n = rows2_n + 1;
    fp.over1_list = over1_list;
    fp.over1_out = over1_out;
    fp.over1_n = over1_n;
  }
  if (no_ws) {
    fp.prefix = 0;  // no floor: visited is the stop position from 0
    all_rows_continue_kernel<<<(unsigned)ceil_div(rows_max, 256), 256, 0, s>>>(row_user, rows_max, cont, cont_n, t0);
    SIMDEX_LAUNCH_CHECK("all_rows_continue");
  } else if ((rc = launch_finalize(fp, rows_max, "finalize_prefix", s))) {
    return rc;
  }
  if (!stage2) {  // the prefix was the whole list
    record_ws_stats(nq, nullptr, 0, bp, ni, f);
    return record_stat_block(ctx, statblk, s);
  }

  // ---- stage 2: continuing users x the whole catalogue.  Buffers are sized
  // for every row; the row and unit counts are read on the device; the count
  // reaches the host statistics slot asynchronously.
  // (slot 0 holds the int32 count in its low half; the high half stays 0)
  if (stats) {
    SIMDEX_CUDA(cudaMemcpyAsync(&host[0], cont_n, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
    SIMDEX_CUDA(cudaStreamSynchronize(s));
    std::vector<int32_t> hc(rows_max);
    SIMDEX_CUDA(cudaMemcpy(hc.data(), st.cnt, sizeof(int32_t) * rows_max, cudaMemcpyDeviceToHost));
    std::vector<int64_t> hu(rows_max);
    SIMDEX_CUDA(cudaMemcpy(hu.data(), row_user, sizeof(int64_t) * rows_max, cudaMemcpyDeviceToHost));
    int64_t tot = 0, live = 0, mx = 0, hist[8] = {0};
    for (int64_t r = 0; r < rows_max; ++r)
      if (hu[r] >= 0) {
        tot += hc[r];
        ++live;
        mx = hc[r] > mx ? hc[r] : mx;
        hist[hc[r] < 16 ? 0 : hc[r] < 32 ? 1 : hc[r] < 64 ? 2 : 3]++;
      }
    fprintf(stderr,
            "[simdex] query_ws nq=%lld continue_past_B=%lld stage1 candidates mean=%.2f max=%lld "
            "<16:%lld <32:%lld <64:%lld >=64:%lld\n",
            (long long)nq, (long long)host[0], live ? (double)tot / live : 0.0, (long long)mx, (long long)hist[0],
            (long long)hist[1], (long long)hist[2], (long long)hist[3]);
  }
  if (list2) {
    // continuing rows grouped by cluster, each cluster's range 128-padded
    SIMDEX_CUDA(cudaMemsetAsync(cnt2, 0, sizeof(int32_t) * c, s));
    SIMDEX_CUDA(cudaMemsetAsync(cur2, 0, sizeof(int32_t) * c, s));
    SIMDEX_CUDA(cudaMemsetAsync(user2, 0xff, sizeof(int64_t) * rows_s2, s));  // padding rows: no user
    cont_count_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows2, 256), 4 * sm_count()), 256, 0, s>>>(
        cont, cont_n, rclus, cnt2);
    SIMDEX_LAUNCH_CHECK("cont_count");
    count_scan_kernel<<<1, 1024, 0, s>>>(cnt2, c, q_off2);
    SIMDEX_LAUNCH_CHECK("count_scan");
    // units: each cluster's rows x its list from B' (list order, stop bounds per tile)
    ws_units_kernel<<<1, 1024, 0, s>>>(q_off2, c, bf_pad, ni - bp, a_off2, units_s2, n_units_s2, bp, rows2_n);
    SIMDEX_LAUNCH_CHECK("ws_units");
    cont_group_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows2, 256), 8 * sm_count()), 256, 0, s>>>(
        cont, cont_n, row_user, row_out, rclus, cu, t0, a_pk, kp, a_off2, cur2, a2, cu2, t02, user2, out2, clus2);
    SIMDEX_LAUNCH_CHECK("cont_group");
    CUtensorMap ma2, mb2;
    if ((rc = make_map(&ma2, a2, rows_s2, kp))) return rc;
    if ((rc = make_map(&mb2, full_b, (int64_t)c * bf_pad, kp))) return rc;
    TopkParams p2 = make_params(st, units_s2, n_units_s2, fnrm, fnmax, cu2, g, f, k_eff);
    p2.row_T0 = t02;
    p2.norm_sorted = 1;
    p2.exit_c = exit_c2;
    p2.exit_m = exit_m2;
    p2.pairs_out = pairs + 1;
    grid = (int)(units_max < g.ctas_per_sm * sm_count() ? units_max : g.ctas_per_sm * sm_count());
    if ((rc = launch_gemm(ma2, mb2, p2, g, grid, "gemm_topk_full", s))) return rc;
    FinalizeParams f2 = fp;
    f2.mode = kFullList;
    f2.total_rows = rows_s2;
    f2.n_rows_dev = rows2_n;
    f2.row_user = user2;
    f2.row_out = out2;
    f2.row_cluster = clus2;
    f2.cont_list = nullptr;
    f2.cont_n = nullptr;
    f2.item_perm = nullptr;
    f2.list_off = bp;
    f2.merge_prefix = 1;
    f2.over1_list = nullptr;
    f2.over1_out = nullptr;
    f2.over1_n = nullptr;
    if ((rc = launch_finalize(f2, rows_s2, "finalize_full", s))) return rc;
    if ((rc = record_stat_block(ctx, statblk, s))) return rc;
    record_ws_stats(nq, &host[0], -1, bp, ni, f);
    // band overflow (rare): exact float64 scan and the visited closed form, for
    // the catalogue-pass rows and for the prefix rows that overflowed
    if ((rc = exact_topk_devcount(users, users32, items, items32, ni, f, over_list, user2, over_n, k, over_out,
                                  out_ids, out_scores, slab, s)))
      return rc;
    fallback_visited_kernel<<<kFallbackGrid, 256, 0, s>>>(over_list, over_n, user2, out2, clus2, list_pos, bounds,
                                                          unorm, ni, bp, k_eff, out_ids, out_scores, out_visited);
    SIMDEX_LAUNCH_CHECK("fallback_visited");
    if ((rc = exact_topk_devcount(users, users32, items, items32, ni, f, over1_list, row_user, over1_n, k, over1_out,
                                  out_ids, out_scores, slab, s)))
      return rc;
    fallback_visited_kernel<<<kFallbackGrid, 256, 0, s>>>(over1_list, over1_n, row_user, row_out, rclus, list_pos,
                                                          bounds, unorm, ni, bp, k_eff, out_ids, out_scores,
                                                          out_visited);
    SIMDEX_LAUNCH_CHECK("fallback_visited");
    return SIMDEX_OK;
  }
  cont_rows_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows2, 32), 8 * sm_count()), 256, 0, s>>>(
      cont, cont_n, rows2, row_user, row_out, rclus, cu, t0, a_pk, kp, a2, cu2, t02, user2, out2, clus2);
  SIMDEX_LAUNCH_CHECK("cont_rows");
  // few continuing rows: catalogue segments spread them over the CTAs
  const bool split = !stats && !getenv("SIMDEX_NO_SPLIT");
  const int64_t units2_cap = units_max > units2 ? units_max : units2;
  units_from_count_kernel<<<(unsigned)ceil_div(units2_cap, 256), 256, 0, s>>>(
      cont_n, 0, ni, split ? units_raw : units_s2, split ? n_units_raw : n_units_s2, units2_cap,
      split ? seg_n : nullptr,
      (int64_t)g.ctas_per_sm * sm_count(), rows_max);
  SIMDEX_LAUNCH_CHECK("units");
  if (!reuse) {  // the catalogue's scaled norms: part of the reusable setup
    item_nrm_kernel<<<(unsigned)ceil_div(ni_pad / 32, 8), 256, 0, s>>>(i_norm, ni, ni_pad, std::ldexp(1.0, si),
                                                                        inrm, inmax);
    SIMDEX_LAUNCH_CHECK("item_nrm");
  }
  CUtensorMap ma2, mb2;
  if ((rc = make_map(&ma2, a2, rows2, kp))) return rc;
  if ((rc = make_map(&mb2, ib, ni_pad, kp))) return rc;
  TopkParams p2 = make_params(st, units_s2, n_units_s2, inrm, inmax, cu2, g, f, k_eff);
  p2.row_T0 = t02;
  p2.norm_sorted = item_perm != nullptr && !getenv("SIMDEX_NO_EARLY_EXIT");
  if (split) {
    SIMDEX_CUDA(cudaMemsetAsync(n_units_s2, 0, sizeof(int32_t), s));
    if (p2.norm_sorted) {
      prune_units_kernel<<<(unsigned)std::min<int64_t>(ceil_div(units2_cap, 8), 8 * sm_count()), 256, 0, s>>>(
          units_raw, n_units_raw, units_s2, n_units_s2, cu2, t02, inmax, p2.g_mul, p2.e_abs, st.cnt, st.flags,
          st.rowT);
    } else {  // no bound to prune with: keep every unit
      prune_units_kernel<<<(unsigned)std::min<int64_t>(ceil_div(units2_cap, 8), 8 * sm_count()), 256, 0, s>>>(
          units_raw, n_units_raw, units_s2, n_units_s2, cu2, t02, inmax, 0.f, INFINITY, st.cnt, st.flags, st.rowT);
    }
    SIMDEX_LAUNCH_CHECK("prune_units");
  }
  p2.pairs_out = pairs + 1;
  Scratch<int64_t> hops2;
  if (stats) {
    SIMDEX_CUDA(hops2.alloc(rows2, s));
    SIMDEX_CUDA(cudaMemsetAsync(hops2.p, 0, sizeof(int64_t) * rows2, s));
    p2.heap_ops = hops2.p;
  }
  grid = (int)(units2_cap < g.ctas_per_sm * sm_count() ? units2_cap : g.ctas_per_sm * sm_count());
  if ((rc = launch_gemm(ma2, mb2, p2, g, grid, "gemm_topk_full", s))) return rc;
  if (split) {
    // (segments exist only for fewer than ~19k continuing rows: a small grid-stride grid)
    merge_segments_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows2, 8), 8 * sm_count()), 256, 0, s>>>(
        cont_n, seg_n, st.cap, st.cid, st.hi, st.cnt, st.flags, st.rowT);
    SIMDEX_LAUNCH_CHECK("merge_segments");
  }
  if (stats) {
    std::vector<int64_t> hh(rows2);
    SIMDEX_CUDA(cudaMemcpy(hh.data(), hops2.p, sizeof(int64_t) * rows2, cudaMemcpyDeviceToHost));
    int64_t tot = 0;
    for (auto v : hh) tot += v;
    fprintf(stderr, "[simdex] stage2 appends per continuing query %.2f\n",
            (double)tot / (double)(host[0] > 0 ? host[0] : 1));
  }
  FinalizeParams f2 = fp;
  f2.mode = kFullList;
  f2.total_rows = rows2;
  f2.n_rows_dev = cont_n;
  f2.row_user = user2;
  f2.row_out = out2;
  f2.row_cluster = clus2;
  f2.cont_list = nullptr;
  f2.cont_n = nullptr;
  f2.item_perm = item_perm;
  if ((rc = launch_finalize(f2, rows2, "finalize_full", s))) return rc;
  if ((rc = record_stat_block(ctx, statblk, s))) return rc;
  record_ws_stats(nq, &host[0], -1, bp, ni, f);
  // band overflow on the full list (rare): exact float64 scan for those users
  // and the same visited closed form; counts read on the device
  if ((rc = exact_topk_devcount(users, users32, items, items32, ni, f, over_list, user2, over_n, k, over_out, out_ids,
                                out_scores, slab, s)))
    return rc;
  fallback_visited_kernel<<<kFallbackGrid, 256, 0, s>>>(over_list, over_n, user2, out2, clus2, list_pos, bounds, unorm,
                                                        ni, bp, k_eff, out_ids, out_scores, out_visited);
  SIMDEX_LAUNCH_CHECK("fallback_visited");
  return SIMDEX_OK;
}

// k-means finalize, a thread per point: the certified candidates' exact
// float64 d2 = (p2 + c2) - 2 p.c (factors in order -- the arithmetic of the
// squared norms, so a point equal to a centre gets exactly 0), first minimum
// (clustering.py:100 + argmin).  Rows whose band overflowed (or, defensively,
// kept no candidate) go to the float64 SIMT pass.
template <class P>
__global__ void __launch_bounds__(256) assign_finalize_kernel(const FinalizeParams p, const P* __restrict__ pts) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  bool changed = false;
  if (r < p.total_rows) {
    bool over = p.row_flags[r] != 0;
    double bd = DBL_MAX;
    int32_t bj = INT32_MAX;
    if (!over) {
      const int cnt = p.row_count[r];
      const float Tr = p.row_T[r];
      const int32_t* cid = p.cand_id + r * p.cap;
      const float* chi = p.cand_hi + r * p.cap;
      const double pp = p.p2[r];
      const P* u = pts + r * p.f;
      for (int e = 0; e < cnt; ++e) {
        if (!(chi[e] >= Tr)) continue;
        const int32_t j = cid[e];
        const double* x = p.items + (int64_t)j * p.f;
        double dot = 0.0;
#pragma unroll 10
        for (int q = 0; q < p.f; ++q) dot = fma(x[q], (double)u[q], dot);
        double d = (pp + p.c2[j]) - 2.0 * dot;
        d = d > 0.0 ? d : 0.0;
        if (d < bd || (d == bd && j < bj)) {
          bd = d;
          bj = j;
        }
      }
      over = bj == INT32_MAX;
    }
    if (over) {
      const int sl = atomicAdd(p.over_n, 1);
      p.over_list[sl] = r;
      p.over_out[sl] = r;
    } else {
      p.out_assign[r] = bj;
      p.out_d2[r] = bd;
      changed = p.prev && p.prev[r] != bj;
    }
  }
  const unsigned m = __ballot_sync(0xffffffffu, changed);
  if (m && lane == __ffs(m) - 1) atomicAdd(p.changed, (unsigned long long)__popc(m));
}

// k-means assignment on the tensor cores (clustering.py:96-101, 175-177):
// augmented product + certified top-1 band, exact float64 d2 over the band's
// candidates.  Rows whose band overflows are returned in over_rows (count in
// *n_over) for the float64 SIMT kernel.  Needs f + 1 <= 256.
template <class P>
int gemm_assign_impl(const double* points, const P* px, const float* points32, int64_t n, int32_t f,
                     P2Fill fill_p2, const double** p2_out, const double* centers, const double* c2, int32_t c,
                     const int64_t* prev, int64_t* out_assign, double* out_d2, unsigned long long* changed,
                     int64_t* over_rows, int32_t* n_over, cudaStream_t s) {
  const int kp = ((f + 1 + 63) / 64) * 64;
  GemmGeometry g;
  int rc = geometry(kp, &g);
  if (rc) return rc;
  const int64_t nu_pad = ceil_div(n, 256) * 256, nc_pad = ceil_div(c, 256) * 256;
  const int64_t nunits = nu_pad / kUnitRows;
  const int k_eff = 1;
  Ctx* ctx = ctx_or_default(nullptr);
  // The point side of the product (squared norms, scale, packed operand,
  // bands, unit list) depends on the points only.  A caller that runs several
  // assignments over the same points (Lloyd iterations) tags the context with
  // a token (simdex_ctx_set_query_token); a call that finds the arena still
  // holding that token's point side -- no other call has used the context
  // since, the arena has not moved, same pointers and sizes -- skips it
  // (0.1 ms of 0.65 per iteration at cfg2).
  const CtxSetup held_before = *ctx_setup(ctx);
  const int64_t qtok = ctx_setup(ctx)->query_token;
  ctx_setup(ctx)->query_token = 0;  // consumed by this call
  uint64_t sig = 1469598103934665603ull;
  for (uint64_t v : {(uint64_t)(uintptr_t)px, (uint64_t)n, (uint64_t)f, (uint64_t)c, (uint64_t)kp,
                     (uint64_t)sizeof(P), (uint64_t)0x6b6d65616e73ull})
    sig = (sig ^ v) * 1099511628211ull;
  Workspace ws(ctx, s);
  unsigned long long* mx;
  int* sexp;
  double* sfac;
  RowState st;
  uint16_t *ua, *ca;
  double *un, *cn, *p2w;
  Unit* units;
  int32_t *n_units, *over_n;
  float *cu, *inrm, *inmax;
  int64_t* over_out;
  ws.add(&mx, 3);
  ws.add(&sexp, 2);
  ws.add(&sfac, 2);
  ws.add(&p2w, nu_pad);
  st.add(ws, nu_pad, k_eff);
  ws.add(&ua, (size_t)nu_pad * kp);
  ws.add(&ca, (size_t)nc_pad * kp);
  ws.add(&un, nu_pad);
  ws.add(&cn, nc_pad);
  ws.add(&units, nunits);
  ws.add(&n_units, 1);
  ws.add(&over_n, 1);
  ws.add(&over_out, n);
  ws.add(&cu, nu_pad);
  ws.add(&inrm, nc_pad);
  ws.add(&inmax, nc_pad / 32);
  if ((rc = ws.commit())) return rc;
  const bool reuse = qtok != 0 && held_before.held_token == qtok && held_before.held_gen == ctx_arena_gen(ctx) &&
                     held_before.held_sig == sig && !getenv("SIMDEX_NO_SETUP_REUSE");
  const double* p2 = p2w;
  *p2_out = p2w;
  SIMDEX_CUDA(cudaMemsetAsync(mx + (reuse ? 1 : 0), 0, (reuse ? 2 : 3) * sizeof(unsigned long long), s));
  const int64_t nf = n * (int64_t)f;
  if (!reuse) {
    if ((rc = fill_p2(px, n, f, p2w, s))) return rc;
    max_abs_any_kernel<P><<<(unsigned)std::min<int64_t>(ceil_div(nf, 256), 4 * 148), 256, 0, s>>>(px, nf, 1.0, mx);
  }
  max_abs_any_kernel<double><<<(unsigned)std::min<int64_t>(ceil_div((int64_t)c * f, 256), 64), 256, 0, s>>>(
      centers, (int64_t)c * f, 1.0, mx + 1);
  max_abs_any_kernel<double><<<1, 256, 0, s>>>(c2, c, 0.5, mx + 2);
  SIMDEX_LAUNCH_CHECK("max_abs_any");
  assign_scales_kernel<<<1, 32, 0, s>>>(mx, eps_for(kp), sexp, sfac);
  SIMDEX_LAUNCH_CHECK("assign_scales");
  ProfileScope _prof("assign_pack", s);
  if (!reuse)
    pack_aug_kernel<P><<<(unsigned)ceil_div(nu_pad * 8, 256), 256, 0, s>>>(px, p2, n, f, 0, sexp, nu_pad, kp,
                                                                            ua, un);
  pack_aug_kernel<double><<<(unsigned)ceil_div(nc_pad * 8, 256), 256, 0, s>>>(centers, c2, c, f, 1, sexp + 1,
                                                                               nc_pad, kp, ca, cn);
  _prof.end();
  SIMDEX_LAUNCH_CHECK("pack_aug");
  if (!reuse) {
    units_from_count_kernel<<<(unsigned)ceil_div(nunits, 256), 256, 0, s>>>(nullptr, n, c, units, n_units, nunits);
    SIMDEX_LAUNCH_CHECK("units");
    row_cu_kernel<<<(unsigned)ceil_div(nu_pad, 256), 256, 0, s>>>(un, n, nu_pad, 0.0, cu, sfac);
    SIMDEX_LAUNCH_CHECK("row_cu");
  }
  if (qtok != 0) {  // the arena now holds this token's point side
    CtxSetup* cs = ctx_setup(ctx);
    cs->held_token = qtok;
    cs->held_gen = ctx_arena_gen(ctx);
    cs->held_sig = sig;
  }
  item_nrm_kernel<<<(unsigned)ceil_div(nc_pad / 32, 8), 256, 0, s>>>(cn, c, nc_pad, 0.0, inrm, inmax,
                                                                      sfac + 1);
  SIMDEX_LAUNCH_CHECK("item_nrm");
  CUtensorMap ma, mb;
  if ((rc = make_map(&ma, ua, nu_pad, kp))) return rc;
  if ((rc = make_map(&mb, ca, nc_pad, kp))) return rc;
  TopkParams tp = make_params(st, units, n_units, inrm, inmax, cu, g, f + 1, k_eff);
  const int grid = (int)(nunits < g.ctas_per_sm * sm_count() ? nunits : g.ctas_per_sm * sm_count());
  if ((rc = launch_gemm(ma, mb, tp, g, grid, "gemm_assign", s))) return rc;
  SIMDEX_CUDA(cudaMemsetAsync(over_n, 0, sizeof(int32_t), s));
  FinalizeParams fp{};
  fp.mode = kAssign;
  fp.total_rows = n;
  fp.nu = n;
  fp.users = points;
  fp.users32 = points32;
  fp.items = centers;
  fp.f = f;
  fp.n = c;
  fp.k_eff = k_eff;
  fp.cap = st.cap;
  fp.cand_id = st.cid;
  fp.cand_hi = st.hi;
  fp.row_T = st.rowT;
  fp.row_count = st.cnt;
  fp.row_flags = st.flags;
  fp.over_list = over_rows;
  fp.over_out = over_out;
  fp.over_n = over_n;
  fp.pow2 = pow2_at_least(std::min(st.cap, std::max(64, 2 * k_eff + 32)));
  fp.p2 = p2;
  fp.c2 = c2;
  fp.prev = prev;
  fp.out_assign = out_assign;
  fp.out_d2 = out_d2;
  fp.changed = changed;
  ProfileScope _pf("finalize_assign", s);
  assign_finalize_kernel<P><<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(fp, px);
  _pf.end();
  SIMDEX_LAUNCH_CHECK("finalize_assign");
  SIMDEX_CUDA(cudaMemcpyAsync(n_over, over_n, sizeof(int32_t), cudaMemcpyDeviceToDevice, s));
  return SIMDEX_OK;
}

int gemm_kmeans_assign(const double* points, const float* points32, int64_t n, int32_t f, P2Fill fill_p2,
                       const double** p2_out, const double* centers, const double* c2, int32_t c,
                       const int64_t* prev, int64_t* out_assign, double* out_d2, unsigned long long* changed,
                       int64_t* over_rows, int32_t* n_over, cudaStream_t s) {
  if (points32)
    return gemm_assign_impl<float>(points, points32, points32, n, f, fill_p2, p2_out, centers, c2, c, prev,
                                   out_assign, out_d2, changed, over_rows, n_over, s);
  return gemm_assign_impl<double>(points, points, nullptr, n, f, fill_p2, p2_out, centers, c2, c, prev, out_assign,
                                  out_d2, changed, over_rows, n_over, s);
}

}  // namespace simdex
