// k-means on device (clustering.py:96-198):
//   * assignment: fused float64 distance GEMM + first-minimum argmin
//     (the U x C distance matrix never reaches HBM, clustering.py:175-177);
//   * update: users ordered by (cluster, id) with the segmented sort, then
//     one CTA per cluster sums its members with a fixed partition and a fixed
//     combination order (deterministic, clustering.py:169-172);
//   * k-means++ seeding with the host's RNG draws: per pass a fused D^2
//     update + block sums, then a one-CTA parallel scan that finds the first
//     index whose cumulative D^2 exceeds u * total (numpy's choice(n, p) ==
//     searchsorted(cumsum(p)/cdf[-1], u, 'right'), clustering.py:118-121).
// Every kernel reads the points either as float64 or, when the caller passes
// an exact float32 copy (all BASELINE inputs are float32 upcast), as float32
// converted back to float64 exactly: same arithmetic, half the bytes.
#include <cfloat>

#include "common.cuh"
#include "sm100.cuh"

namespace simdex {

int gemm_kmeans_assign(const double* points, const float* points32, int64_t n, int32_t f, const double* p2,
                       const double* centers, const double* c2, int32_t c, const int64_t* prev, int64_t* out_assign,
                       double* out_d2, unsigned long long* changed, int64_t* over_rows, int32_t* n_over,
                       cudaStream_t s);

namespace {

constexpr int kAssignGemmMaxF = 256;  // augmented K (f + 1) the tensor-core path takes
constexpr int kAssignThreads = 128;
constexpr int kCC = 32;  // centers per chunk (register accumulators)
constexpr int kFC = 32;  // factors per chunk

template <class P>
__global__ void sqnorm_kernel(const P* __restrict__ x, int64_t n, int f, double* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int k = 0; k < f; ++k) {
    const double v = (double)x[i * f + k];
    s = fma(v, v, s);
  }
  out[i] = s;
}

template <class P>
__global__ void __launch_bounds__(kAssignThreads) assign_kernel(
    const P* __restrict__ points, const double* __restrict__ p2, int64_t n, int f, const double* __restrict__ centers,
    const double* __restrict__ c2, int c, const int64_t* __restrict__ prev, int64_t* __restrict__ out_assign,
    double* __restrict__ out_d2, unsigned long long* __restrict__ changed, double* __restrict__ block_sums,
    const int64_t* __restrict__ rows, int64_t n_rows) {
  __shared__ double cs[kCC][kFC + 1];
  __shared__ double red[kAssignThreads / 32];
  const int64_t idx = (int64_t)blockIdx.x * kAssignThreads + threadIdx.x;
  const bool live = rows ? idx < n_rows : idx < n;
  const int64_t u = rows ? (live ? rows[idx] : 0) : idx;
  const P* x = points + (live ? u : 0) * f;
  const double pp = live ? p2[u] : 0.0;
  double best = DBL_MAX;
  int64_t arg = 0;
  for (int c0 = 0; c0 < c; c0 += kCC) {
    double acc[kCC];
#pragma unroll
    for (int j = 0; j < kCC; ++j) acc[j] = 0.0;
    for (int k0 = 0; k0 < f; k0 += kFC) {
      __syncthreads();
      for (int e = threadIdx.x; e < kCC * kFC; e += kAssignThreads) {
        int j = e / kFC, k = e % kFC;
        cs[j][k] = (c0 + j < c && k0 + k < f) ? centers[(int64_t)(c0 + j) * f + k0 + k] : 0.0;
      }
      __syncthreads();
      const int kn = (f - k0) < kFC ? (f - k0) : kFC;
      for (int k = 0; k < kn; ++k) {
        const double xk = live ? (double)x[k0 + k] : 0.0;
#pragma unroll
        for (int j = 0; j < kCC; ++j) acc[j] = fma(xk, cs[j][k], acc[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < kCC; ++j) {
      if (c0 + j < c) {
        double d = (pp + c2[c0 + j]) - 2.0 * acc[j];  // clustering.py:100
        d = d > 0.0 ? d : 0.0;                        // np.maximum(d2, 0)
        if (d < best) {                               // strict: first minimum wins (argmin)
          best = d;
          arg = c0 + j;
        }
      }
    }
  }
  double mine = 0.0;
  if (live) {
    out_assign[u] = arg;
    out_d2[u] = best;
    mine = best;
    if (prev && prev[u] != arg) atomicAdd(changed, 1ull);
  }
  mine = warp_sum(mine);  // deterministic block sum of d2 (fixed tree)
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kAssignThreads / 32; ++w) s += red[w];
    if (block_sums) block_sums[blockIdx.x] = s;
  }
}

// per-block sums of x (fixed tree): the objective from out_d2
__global__ void block_sum_kernel(const double* __restrict__ x, int64_t n, double* __restrict__ part) {
  __shared__ double red[8];
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  double v = i < n ? x[i] : 0.0;
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < 8; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

// Sum `m` partials in a fixed order (one CTA).
__global__ void sum_partials_kernel(const double* __restrict__ part, int64_t m, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) s += part[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t;
  }
}

__global__ void cluster_keys_kernel(const int64_t* __restrict__ assign, int64_t n, double* keys, int32_t* ids,
                                    unsigned long long* counts) {
  int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  keys[u] = -(double)assign[u];  // sort desc on -cluster == cluster ascending, then id ascending
  ids[u] = (int32_t)u;
  atomicAdd(counts + assign[u], 1ull);
}

__global__ void offsets_kernel(const unsigned long long* counts, int c, int64_t* out_counts, int64_t* offsets) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  int64_t acc = 0;
  for (int j = 0; j < c; ++j) {
    offsets[j] = acc;
    out_counts[j] = (int64_t)counts[j];
    acc += (int64_t)counts[j];
  }
  offsets[c] = acc;
}

__global__ void members_kernel(const int32_t* ids, int64_t n, int64_t* members) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) members[i] = ids[i];
}

// One CTA (8 warps) per cluster: warp w sums members w, w+8, ... with its
// lanes on consecutive factors (coalesced row reads), then the 8 warp partials
// are added in warp order.  Fixed partition and order: deterministic.  Empty
// clusters keep their centroid (clustering.py:170-172).
constexpr int kMeanWarps = 8;
constexpr int kMeanRegs = 4;  // factors per lane per chunk (128-factor chunks)

template <class P>
__global__ void __launch_bounds__(kMeanWarps * 32) centroid_mean_kernel(const P* __restrict__ points, int f,
                                                                        const int64_t* __restrict__ members,
                                                                        const int64_t* __restrict__ offsets,
                                                                        double* __restrict__ centers) {
  __shared__ double part[kMeanWarps][kMeanRegs * 32];
  const int c = blockIdx.x;
  const int64_t b = offsets[c], e = offsets[c + 1];
  if (e == b) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k0 = 0; k0 < f; k0 += kMeanRegs * 32) {
    double acc[kMeanRegs];
#pragma unroll
    for (int q = 0; q < kMeanRegs; ++q) acc[q] = 0.0;
    int64_t m = b + w;
    for (; m + 3 * kMeanWarps < e; m += 4 * kMeanWarps) {  // 4 independent rows in flight
      const P* r0 = points + members[m] * f + k0;
      const P* r1 = points + members[m + kMeanWarps] * f + k0;
      const P* r2 = points + members[m + 2 * kMeanWarps] * f + k0;
      const P* r3 = points + members[m + 3 * kMeanWarps] * f + k0;
#pragma unroll
      for (int q = 0; q < kMeanRegs; ++q) {
        const int k = lane + 32 * q;
        if (k0 + k < f) {
          const double v0 = (double)r0[k], v1 = (double)r1[k], v2 = (double)r2[k], v3 = (double)r3[k];
          acc[q] = (((acc[q] + v0) + v1) + v2) + v3;
        }
      }
    }
    for (; m < e; m += kMeanWarps) {
      const P* r0 = points + members[m] * f + k0;
#pragma unroll
      for (int q = 0; q < kMeanRegs; ++q) {
        const int k = lane + 32 * q;
        if (k0 + k < f) acc[q] += (double)r0[k];
      }
    }
#pragma unroll
    for (int q = 0; q < kMeanRegs; ++q) part[w][lane + 32 * q] = acc[q];
    __syncthreads();
    for (int k = threadIdx.x; k < kMeanRegs * 32 && k0 + k < f; k += blockDim.x) {
      double tot = 0.0;
#pragma unroll
      for (int ww = 0; ww < kMeanWarps; ++ww) tot += part[ww][k];
      centers[(int64_t)c * f + k0 + k] = tot / (double)(e - b);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// k-means++ seeding
// ---------------------------------------------------------------------------
constexpr int kSeedThreads = 256;
constexpr int kPickThreads = 1024;

// d2 = min(d2, |p - center_j|^2) with the reference's expression
// (||p||^2 + ||c||^2 - 2 p.c, clipped); pass 0 initialises.  Also block sums.
// Points whose nearest seed a is far from the new center skip the distance:
// |c_j - c_a|^2 >= 4 (d2 + eta)(1 + 2^-30), eta = 2^-40 (p2 + c2_j + c2_a)
// bounds the float64 cancellation of the expression, so by the triangle
// inequality the computed distance could not go below d2 and min() would keep
// d2: the skip is bit-exact.  Each warp owns 32 consecutive points; the ones
// that need the distance are taken 4 at a time, 8 lanes per point on strided
// factors (coalesced row reads, all loads issued before the FMAs), reduced by
// a fixed shuffle tree; the block sum adds the points in a fixed order.
constexpr int kSeedWarps = kSeedThreads / 32;
constexpr int kSeedBufBytes = 16384;  // per-warp row staging cap

struct SeedSmem {  // dynamic shared layout of seed_update_kernel
  int batch;       // rows staged per bulk copy (<= 32)
  size_t buf;      // bytes per warp buffer
  size_t cen_off, bar_off, buf_off, total;
};

__host__ __device__ inline SeedSmem seed_smem(int f, size_t esize) {
  SeedSmem m;
  const size_t row = (size_t)f * esize;
  int b = (int)(kSeedBufBytes / row);
  m.batch = b > 32 ? 32 : (b < 1 ? 1 : b);
  m.buf = (((size_t)m.batch * row + 32) + 127) & ~size_t(127);
  m.cen_off = 0;
  m.bar_off = ((size_t)f * 8 + 15) & ~size_t(15);
  m.buf_off = (m.bar_off + kSeedWarps * 8 + 127) & ~size_t(127);
  m.total = m.buf_off + kSeedWarps * m.buf;
  return m;
}

template <class P>
__global__ void __launch_bounds__(kSeedThreads, 4) seed_update_kernel(const P* __restrict__ points,
                                                                   const double* __restrict__ p2, int64_t n, int f,
                                                                   const int64_t* __restrict__ rows, int j,
                                                                   double* __restrict__ d2,
                                                                   int32_t* __restrict__ near,
                                                                   const double* __restrict__ seed_c2,
                                                                   const double* __restrict__ cd2,
                                                                   double* __restrict__ block_sums,
                                                                   const int32_t* __restrict__ degenerate) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  __shared__ double red[kSeedWarps];
  if (*degenerate >= 0) return;
  const SeedSmem L = seed_smem(f, sizeof(P));
  double* cen = reinterpret_cast<double*>(sm_raw + L.cen_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_raw + L.bar_off);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, sl = lane & 7, grp = lane >> 3;
  unsigned char* buf = sm_raw + L.buf_off + w * L.buf;
  const int64_t wbase = (int64_t)blockIdx.x * kSeedThreads + w * 32;
  const int64_t me = wbase + lane;
  const size_t row_bytes = (size_t)f * sizeof(P);
  const size_t total_bytes = (size_t)n * row_bytes;
  const unsigned char* gbase = reinterpret_cast<const unsigned char*>(points);
  if (lane == 0) {
    sm100::mbar_init(bars + w, 1);
    sm100::fence_barrier_init();
  }
  double old = DBL_MAX, mp2 = 0.0;
  int a = 0;
  if (me < n) {
    mp2 = p2[me];
    if (j > 0) {
      old = d2[me];
      a = near[me];
    }
  }
  const int64_t r = rows[j];
  for (int k = threadIdx.x; k < f; k += kSeedThreads) cen[k] = (double)points[r * f + k];
  __syncthreads();
  const double cc = p2[r];
  bool need = me < n;
  if (need && j > 0) {
    const double eta = 0x1p-40 * (mp2 + cc + seed_c2[a]);
    need = !(cd2[a] >= 4.0 * (old + eta) * (1.0 + 0x1p-30));
  }
  double fin = old;  // this lane's point's d2 after the pass
  const unsigned needm = __ballot_sync(0xffffffffu, need);
  uint32_t phase = 0;
  for (int b0 = 0; b0 < 32; b0 += L.batch) {
    const unsigned bm = L.batch >= 32 ? 0xffffffffu : (((1u << L.batch) - 1u) << b0);
    unsigned pend = needm & bm;
    if (!pend) continue;
    // stage the batch's contiguous rows in shared memory with one bulk copy
    const int64_t u0 = wbase + b0;
    const int64_t u1 = (wbase + b0 + L.batch) < n ? (wbase + b0 + L.batch) : n;
    const size_t start = (size_t)u0 * row_bytes, a0 = start & ~size_t(15);
    const size_t sz = ((size_t)u1 * row_bytes - a0 + 15) & ~size_t(15);
    const bool staged = a0 + sz <= total_bytes;  // else (buffer tail) read the rows from global
    if (staged) {
      __syncwarp();
      if (lane == 0) {
        sm100::fence_proxy_async_smem();
        sm100::mbar_arrive_expect_tx(bars + w, (uint32_t)sz);
        sm100::bulk_load_1d(buf, gbase + a0, (uint32_t)sz, bars + w);
      }
      sm100::mbar_wait(bars + w, phase);
      phase ^= 1;
    }
    const unsigned char* sbase = buf + (start - a0);
    if (need && lane >= b0 && lane < b0 + L.batch) {  // lane per point, row from shared memory
      const P* x = staged ? reinterpret_cast<const P*>(sbase + (size_t)(lane - b0) * row_bytes) : points + me * f;
      double dot = 0.0;
#pragma unroll 5
      for (int k = 0; k < f; ++k) dot = fma((double)x[k], cen[k], dot);
      double d = (mp2 + cc) - 2.0 * dot;
      d = d > 0.0 ? d : 0.0;
      if (j == 0 || d < old) {
        d2[me] = d;
        near[me] = j;
        fin = d;
      }
    }
  }
  double v = me < n ? fin : 0.0;
  v = warp_sum(v);
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int ww = 0; ww < kSeedWarps; ++ww) s += red[ww];
    block_sums[blockIdx.x] = s;
  }
}

// One CTA: pick seed j+1 = first index i with cumsum(d2)[i] > u * total.
// Thread t owns a contiguous run of block sums; runs are combined by a fixed
// in-CTA scan (deterministic); the crossing run, then block, then element
// are located in turn.
template <class P>
__global__ void __launch_bounds__(kPickThreads) seed_pick_kernel(const P* __restrict__ points, int64_t n, int f,
                                                                 const double* __restrict__ d2,
                                                                 const double* __restrict__ block_sums,
                                                                 int64_t nblocks, const double* __restrict__ uniforms,
                                                                 int j, int64_t* __restrict__ rows,
                                                                 double* __restrict__ centers,
                                                                 const double* __restrict__ p2,
                                                                 double* __restrict__ seed_c2,
                                                                 double* __restrict__ cd2,
                                                                 int32_t* __restrict__ degenerate) {
  __shared__ double scan[kPickThreads];
  __shared__ double wsum[kSeedThreads / 32];
  __shared__ int64_t s_block;
  __shared__ double s_base;
  __shared__ unsigned long long s_pick;
  if (*degenerate >= 0) return;
  const int t = threadIdx.x;
  const int64_t per = (nblocks + kPickThreads - 1) / kPickThreads;
  const int64_t b0 = t * per, b1 = (b0 + per) < nblocks ? (b0 + per) : nblocks;
  double mine = 0.0;
  for (int64_t b = b0; b < b1; ++b) mine += block_sums[b];
  scan[t] = mine;
  __syncthreads();
  for (int off = 1; off < kPickThreads; off <<= 1) {  // inclusive Hillis-Steele scan
    const double o = t >= off ? scan[t - off] : 0.0;
    __syncthreads();
    scan[t] += o;
    __syncthreads();
  }
  const double total = scan[kPickThreads - 1];
  if (!(total > 0.0)) {
    if (t == 0) *degenerate = j + 1;
    return;
  }
  const double target = uniforms[j] * total;
  if (t == 0) {
    s_block = -1;
    s_pick = ~0ull;
  }
  __syncthreads();
  const double excl = scan[t] - mine;
  if (b0 < b1 && scan[t] > target && !(excl > target)) {  // the run holding the crossing
    double acc = excl;
    int64_t b = b0;
    for (; b < b1; ++b) {
      if (acc + block_sums[b] > target) break;
      acc += block_sums[b];
    }
    if (b == b1) {  // rounding between the two summation orders: last block of the run
      b = b1 - 1;
      acc = excl;
      for (int64_t q = b0; q < b; ++q) acc += block_sums[q];
    }
    s_block = b;
    s_base = acc;
  }
  __syncthreads();
  if (s_block < 0 && t == 0) {  // target beyond the rounded total: last positive block
    int64_t b = nblocks - 1;
    while (b > 0 && !(block_sums[b] > 0.0)) --b;
    double acc = 0.0;
    for (int64_t q = 0; q < b; ++q) acc += block_sums[q];
    s_block = b;
    s_base = acc;
  }
  __syncthreads();
  const int64_t bb = s_block * kSeedThreads;
  const int lane = t & 31, wid = t >> 5;
  const int64_t i = bb + t;
  double v = 0.0, x = 0.0;
  if (t < kSeedThreads) {  // warp-uniform: the first 8 warps scan the block
    v = i < n ? d2[i] : 0.0;
    x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
  }
  __syncthreads();
  if (t < kSeedThreads) {
    double pre = s_base;
    for (int w = 0; w < wid; ++w) pre += wsum[w];
    const double incl = pre + x;
    if (i < n && v > 0.0 && incl > target && !(incl - v > target)) atomicMin(&s_pick, (unsigned long long)i);
  }
  __syncthreads();
  if (t == 0) {
    int64_t p = s_pick == ~0ull ? -1 : (int64_t)s_pick;
    if (p < 0) {  // defensive: last positive entry of the block
      for (int64_t q = bb + kSeedThreads - 1; q >= bb; --q)
        if (q < n && d2[q] > 0.0) {
          p = q;
          break;
        }
    }
    rows[j + 1] = p;
    s_pick = (unsigned long long)p;
  }
  __syncthreads();
  const int64_t p = (int64_t)s_pick;
  double* cnew = scan;  // reuse: the new center, then squared distances to the earlier seeds
  for (int k = t; k < f; k += blockDim.x) {
    const double v = (double)points[p * f + k];
    centers[(int64_t)(j + 1) * f + k] = v;
    cnew[k] = v;
  }
  if (t == 0) seed_c2[j + 1] = p2[p];
  __syncthreads();
  // squared distances new seed -> seeds 0..j: 4 lanes per seed, 8 seeds per warp
  // per round, all loads of a round in flight together
  const int g4 = lane >> 2, l4 = lane & 3;
  for (int q0 = wid * 8; q0 <= j; q0 += kPickThreads / 4) {
    const int q = q0 + g4;
    double acc = 0.0;
    if (q <= j) {
      const double* cq = centers + (int64_t)q * f;
      for (int k0 = 0; k0 < f; k0 += 64) {
        double xv[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int k = k0 + l4 + 4 * i;
          xv[i] = k < f ? cq[k] : 0.0;
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int k = k0 + l4 + 4 * i;
          if (k < f) {
            const double d = cnew[k] - xv[i];
            acc = fma(d, d, acc);
          }
        }
      }
    }
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (q <= j && l4 == 0) cd2[q] = acc;
  }
}

template <class P>
__global__ void seed_first_kernel(const P* __restrict__ points, int f, int64_t first, int64_t* rows, double* centers,
                                  const double* __restrict__ p2, double* __restrict__ seed_c2, int32_t* degenerate) {
  if (threadIdx.x == 0) {
    rows[0] = first;
    seed_c2[0] = p2[first];
    *degenerate = -1;
  }
  for (int k = threadIdx.x; k < f; k += blockDim.x) centers[k] = (double)points[first * f + k];
}

__global__ void to_f32_kernel(const double* __restrict__ x, int64_t n, float* __restrict__ out,
                              int32_t* __restrict__ inexact) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool bad = false;
  if (i < n) {
    const float v = (float)x[i];
    out[i] = v;
    bad = (double)v != x[i];
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(inexact, 1);
}

// ---------------------------------------------------------------------------
// launchers (float64 or exact float32 points)
// ---------------------------------------------------------------------------
template <class P>
int assign_impl(const double* points, const float* points32, const P* px, int64_t n, int32_t f,
                const double* centers, int32_t c, const int64_t* prev, int64_t* out_assign, double* out_d2,
                int64_t* out_changed, double* out_objective, cudaStream_t s) {
  Scratch<double> p2, c2, part;
  SIMDEX_CUDA(p2.alloc(n, s));
  SIMDEX_CUDA(c2.alloc(c, s));
  sqnorm_kernel<P><<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(px, n, f, p2.p);
  SIMDEX_LAUNCH_CHECK("sqnorm");
  sqnorm_kernel<double><<<(unsigned)ceil_div(c, 256), 256, 0, s>>>(centers, c, f, c2.p);
  SIMDEX_LAUNCH_CHECK("sqnorm");
  SIMDEX_CUDA(cudaMemsetAsync(out_changed, 0, sizeof(int64_t), s));
  auto* changed = reinterpret_cast<unsigned long long*>(out_changed);
  if (f + 1 <= kAssignGemmMaxF) {
    // tensor-core candidates + exact float64 d2; overflowing bands go to the SIMT kernel
    Scratch<int64_t> over;
    SIMDEX_CUDA(over.alloc(n, s));
    int32_t n_over = 0;
    int rc = gemm_kmeans_assign(points, points32, n, f, p2.p, centers, c2.p, c, prev, out_assign, out_d2, changed,
                                over.p, &n_over, s);
    if (rc) return rc;
    if (n_over > 0) {
      assign_kernel<P><<<(unsigned)ceil_div(n_over, kAssignThreads), kAssignThreads, 0, s>>>(
          px, p2.p, n, f, centers, c2.p, c, prev, out_assign, out_d2, changed, nullptr, over.p, n_over);
      SIMDEX_LAUNCH_CHECK("assign");
    }
  } else {
    ProfileScope _prof("kmeans_assign", s);
    assign_kernel<P><<<(unsigned)ceil_div(n, kAssignThreads), kAssignThreads, 0, s>>>(
        px, p2.p, n, f, centers, c2.p, c, prev, out_assign, out_d2, changed, nullptr, nullptr, 0);
    _prof.end();
    SIMDEX_LAUNCH_CHECK("assign");
  }
  const int64_t nb = ceil_div(n, 256);
  SIMDEX_CUDA(part.alloc(nb, s));
  block_sum_kernel<<<(unsigned)nb, 256, 0, s>>>(out_d2, n, part.p);
  SIMDEX_LAUNCH_CHECK("block_sum");
  sum_partials_kernel<<<1, 1024, 0, s>>>(part.p, nb, out_objective);
  SIMDEX_LAUNCH_CHECK("sum_partials");
  return SIMDEX_OK;
}

template <class P>
int seed_impl(const P* points, int64_t n, int32_t f, int32_t k, int64_t first, const double* uniforms,
              int64_t* out_rows, double* out_centers, int32_t* out_deg, cudaStream_t s) {
  if (f > kPickThreads) {
    set_error("kmeans_seed: f > %d", kPickThreads);
    return SIMDEX_EUNSUPPORTED;
  }
  const int64_t nb = ceil_div(n, kSeedThreads);
  Scratch<double> p2, d2, part, seed_c2, cd2;
  Scratch<int32_t> near;
  SIMDEX_CUDA(p2.alloc(n, s));
  SIMDEX_CUDA(d2.alloc(n, s));
  SIMDEX_CUDA(near.alloc(n, s));
  SIMDEX_CUDA(part.alloc(nb, s));
  SIMDEX_CUDA(seed_c2.alloc(k, s));
  SIMDEX_CUDA(cd2.alloc(k, s));
  sqnorm_kernel<P><<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(points, n, f, p2.p);
  SIMDEX_LAUNCH_CHECK("sqnorm");
  seed_first_kernel<P><<<1, 128, 0, s>>>(points, f, first, out_rows, out_centers, p2.p, seed_c2.p, out_deg);
  SIMDEX_LAUNCH_CHECK("seed_first");
  const size_t smem = seed_smem(f, sizeof(P)).total;
  if (smem > 48 * 1024)
    SIMDEX_CUDA(cudaFuncSetAttribute(seed_update_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int j = 0; j + 1 < k; ++j) {
    ProfileScope _prof("seed_update", s);
    seed_update_kernel<P><<<(unsigned)nb, kSeedThreads, smem, s>>>(points, p2.p, n, f, out_rows, j, d2.p, near.p,
                                                                   seed_c2.p, cd2.p, part.p, out_deg);
    _prof.end();
    ProfileScope _prof2("seed_pick", s);
    seed_pick_kernel<P><<<1, kPickThreads, 0, s>>>(points, n, f, d2.p, part.p, nb, uniforms, j, out_rows, out_centers,
                                                   p2.p, seed_c2.p, cd2.p, out_deg);
    _prof2.end();
    count_launches(2);
  }
  SIMDEX_CUDA(cudaGetLastError());
  return SIMDEX_OK;
}

template <class P>
int mean_impl(const P* points, int32_t f, const int64_t* members, const int64_t* offsets, int32_t c,
              double* centers, cudaStream_t s) {
  ProfileScope _prof("centroid_mean", s);
  centroid_mean_kernel<P><<<(unsigned)c, kMeanWarps * 32, 0, s>>>(points, f, members, offsets, centers);
  _prof.end();
  SIMDEX_LAUNCH_CHECK("centroid_mean");
  return SIMDEX_OK;
}

}  // namespace
}  // namespace simdex

using namespace simdex;

extern "C" int simdex_to_f32(const double* x, int64_t n, float* out, int32_t* inexact, void* stream) {
  SIMDEX_CHECK_ARG(x && out && inexact, "simdex_to_f32: null pointer");
  SIMDEX_CHECK_ARG(n >= 0, "simdex_to_f32: bad sizes");
  cudaStream_t s = as_stream(stream);
  SIMDEX_CUDA(cudaMemsetAsync(inexact, 0, sizeof(int32_t), s));
  if (n == 0) return SIMDEX_OK;
  to_f32_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(x, n, out, inexact);
  SIMDEX_LAUNCH_CHECK("to_f32");
  return SIMDEX_OK;
}

extern "C" int simdex_kmeans_assign(const double* points, const float* points32, int64_t n, int32_t f,
                                    const double* centers, int32_t c, const int64_t* prev_assign, int64_t* out_assign,
                                    double* out_d2, int64_t* out_changed, double* out_objective, void* stream) {
  SIMDEX_CHECK_ARG((points || points32) && centers && out_assign && out_d2 && out_changed && out_objective,
                   "simdex_kmeans_assign: null pointer");
  SIMDEX_CHECK_ARG(n >= 1 && f >= 1 && c >= 1, "simdex_kmeans_assign: bad sizes");
  cudaStream_t s = as_stream(stream);
  if (points32)
    return assign_impl<float>(points, points32, points32, n, f, centers, c, prev_assign, out_assign, out_d2,
                              out_changed, out_objective, s);
  return assign_impl<double>(points, nullptr, points, n, f, centers, c, prev_assign, out_assign, out_d2, out_changed,
                             out_objective, s);
}

extern "C" int simdex_kmeans_update(const double* points, const float* points32, int64_t n, int32_t f,
                                    const int64_t* assign, int32_t c, double* centers, int64_t* out_counts,
                                    int64_t* out_members, int64_t* out_offsets, void* stream) {
  SIMDEX_CHECK_ARG((points || points32) && assign && out_counts && out_members && out_offsets,
                   "simdex_kmeans_update: null pointer");
  SIMDEX_CHECK_ARG(n >= 1 && f >= 1 && c >= 1 && n < INT32_MAX, "simdex_kmeans_update: bad sizes");
  cudaStream_t s = as_stream(stream);
  Scratch<double> keys;
  Scratch<int32_t> ids;
  Scratch<unsigned long long> cnt;
  SIMDEX_CUDA(keys.alloc(n, s));
  SIMDEX_CUDA(ids.alloc(n, s));
  SIMDEX_CUDA(cnt.alloc(c, s));
  SIMDEX_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * c, s));
  cluster_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(assign, n, keys.p, ids.p, cnt.p);
  SIMDEX_LAUNCH_CHECK("cluster_keys");
  SIMDEX_CUDA(segmented_sort_desc(keys.p, ids.p, 1, n, s));
  offsets_kernel<<<1, 32, 0, s>>>(cnt.p, c, out_counts, out_offsets);
  SIMDEX_LAUNCH_CHECK("offsets");
  members_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(ids.p, n, out_members);
  SIMDEX_LAUNCH_CHECK("members");
  if (!centers) return SIMDEX_OK;  // grouping only (members/offsets/counts)
  if (points32) return mean_impl<float>(points32, f, out_members, out_offsets, c, centers, s);
  return mean_impl<double>(points, f, out_members, out_offsets, c, centers, s);
}

extern "C" int simdex_kmeans_seed(const double* points, const float* points32, int64_t n, int32_t f, int32_t k,
                                  int64_t first, const double* uniforms, int64_t* out_rows, double* out_centers,
                                  int32_t* out_degenerate_pass, void* stream) {
  SIMDEX_CHECK_ARG((points || points32) && out_rows && out_centers && out_degenerate_pass,
                   "simdex_kmeans_seed: null pointer");
  SIMDEX_CHECK_ARG(n >= 1 && f >= 1 && k >= 1 && k <= n && first >= 0 && first < n,
                   "simdex_kmeans_seed: bad sizes");
  SIMDEX_CHECK_ARG(k == 1 || uniforms, "simdex_kmeans_seed: uniforms required");
  cudaStream_t s = as_stream(stream);
  if (points32)
    return seed_impl<float>(points32, n, f, k, first, uniforms, out_rows, out_centers, out_degenerate_pass, s);
  return seed_impl<double>(points, n, f, k, first, uniforms, out_rows, out_centers, out_degenerate_pass, s);
}
