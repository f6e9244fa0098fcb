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
#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace simdex {

int gemm_kmeans_assign(const double* points, const float* points32, int64_t n, int32_t f, P2Fill fill_p2,
                       const double** p2_out, const double* centers, const double* c2, int32_t c,
                       const int64_t* prev, int64_t* out_assign, double* out_d2, unsigned long long* changed,
                       int64_t* over_rows, int32_t* n_over_dev, cudaStream_t s);

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

// Exact float64 assignment (clustering.py:96-101), one thread per point.
// With `rows` it handles the listed points only (count read on the device,
// grid-stride over blocks so the host needs no count).
template <class P>
__global__ void __launch_bounds__(kAssignThreads) assign_kernel(
    const P* __restrict__ points, const double* __restrict__ p2, int64_t n, int f, const double* __restrict__ centers,
    const double* __restrict__ c2, int c, const int64_t* __restrict__ prev, int64_t* __restrict__ out_assign,
    double* __restrict__ out_d2, unsigned long long* __restrict__ changed, const int64_t* __restrict__ rows,
    const int32_t* __restrict__ n_rows) {
  __shared__ double cs[kCC][kFC + 1];
  const int64_t limit = rows ? (int64_t)*n_rows : n;
  for (int64_t base = (int64_t)blockIdx.x * kAssignThreads; base < limit;
       base += (int64_t)gridDim.x * kAssignThreads) {
    const int64_t idx = base + threadIdx.x;
    const bool live = idx < limit;
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
    if (live) {
      out_assign[u] = arg;
      out_d2[u] = best;
      if (prev && prev[u] != arg) atomicAdd(changed, 1ull);
    }
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

// Cluster c's members are split into S contiguous parts (one CTA each,
// blockIdx.x = c * S + s); part sums go to psum[c][s][f] and are combined in
// part order by combine_mean_kernel.
template <class P>
__global__ void __launch_bounds__(kMeanWarps * 32) centroid_mean_kernel(const P* __restrict__ points, int f,
                                                                        const int64_t* __restrict__ members,
                                                                        const int64_t* __restrict__ offsets, int S,
                                                                        double* __restrict__ psum) {
  __shared__ double part[kMeanWarps][kMeanRegs * 32];
  const int c = blockIdx.x / S, sp = blockIdx.x % S;
  const int64_t cb = offsets[c], ce = offsets[c + 1];
  const int64_t b = cb + (ce - cb) * sp / S, e = cb + (ce - cb) * (sp + 1) / S;
  double* out = psum + ((int64_t)c * S + sp) * f;
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
      out[k0 + k] = tot;
    }
    __syncthreads();
  }
}

// centroid = sum over members in id order / count: the reference's
// users[sel].mean(axis=0) adds the rows in order (numpy reduces a
// non-contiguous axis sequentially), so the centroids are bit-identical to
// the reference's for the same assignment.  One CTA per cluster: member rows
// are staged in shared memory 64 at a time with asynchronous copies (double
// buffered), thread k adds factor k sequentially.  Empty clusters keep their
// centroid (clustering.py:170-172).
constexpr int kSeqMaxF = 1024;  // 8 factors per thread

template <class P>
__global__ void __launch_bounds__(128) centroid_seq_kernel(const P* __restrict__ points, int f,
                                                           const int64_t* __restrict__ members,
                                                           const int64_t* __restrict__ offsets, int kSeqRows,
                                                           double* __restrict__ centers) {
  extern __shared__ __align__(16) unsigned char seq_raw[];
  P* buf = reinterpret_cast<P*>(seq_raw);  // [2][kSeqRows * f]
  __shared__ int64_t ids[256];             // member ids of the chunk being staged
  const int cl = blockIdx.x, t = threadIdx.x;
  const int64_t b = offsets[cl], e = offsets[cl + 1];
  if (e == b) return;
  const int64_t nchunk = (e - b + kSeqRows - 1) / kSeqRows;
  auto rows_of = [&](int64_t ch) {
    const int64_t r0 = b + ch * kSeqRows;
    return (int)((e - r0) < kSeqRows ? (e - r0) : kSeqRows);
  };
  // ids of the chunk in shared memory first, then one asynchronous copy per
  // element with no load on its address path
  auto stage = [&](int64_t ch, int slot) {
    const int rows = rows_of(ch);
    for (int i = t; i < rows; i += blockDim.x) ids[i] = members[b + ch * kSeqRows + i];
    __syncthreads();
    P* dst = buf + (size_t)slot * kSeqRows * f;
    // warp per row, lanes across 8-byte pieces (two floats when f is even)
    const int lane = t & 31, nw = blockDim.x >> 5;
    const bool pairs = sizeof(P) == 4 && (f & 1) == 0;
    const int pieces = pairs ? f >> 1 : f;
    for (int r = t >> 5; r < rows; r += nw) {
      const P* src = points + ids[r] * f;
      P* d = dst + (size_t)r * f;
      for (int q = lane; q < pieces; q += 32) {
        if (pairs)
          sm100::cp_async8(d + 2 * q, src + 2 * q);
        else if constexpr (sizeof(P) == 8)
          sm100::cp_async8(d + q, src + q);
        else
          sm100::cp_async4(d + q, src + q);
      }
    }
    sm100::cp_async_commit();
    __syncthreads();  // ids may be overwritten by the next stage
  };
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // thread t owns factors t + 128 h
  stage(0, 0);
  for (int64_t ch = 0; ch < nchunk; ++ch) {
    sm100::cp_async_wait<0>();  // chunk ch landed
    __syncthreads();
    if (ch + 1 < nchunk) stage(ch + 1, (int)((ch + 1) & 1));  // streams while chunk ch is summed
    const int rows = rows_of(ch);
    const P* src = buf + (size_t)(ch & 1) * kSeqRows * f;
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const int k = t + 128 * h;
      if (k < f) {
#pragma unroll 8
        for (int r = 0; r < rows; ++r) acc[h] += (double)src[r * f + k];
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    const int k = t + 128 * h;
    if (k < f) centers[(int64_t)cl * f + k] = acc[h] / (double)(e - b);
  }
}

// rows in member order: sorted[j] = points[members[j]] (a warp per 8 rows,
// lanes across the row), so every cluster's rows are one contiguous range
template <class P>
__global__ void gather_rows_kernel(const P* __restrict__ points, int f, const int64_t* __restrict__ members,
                                   int64_t n, P* __restrict__ sorted) {
  const int lane = threadIdx.x & 31;
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (int64_t j = w * 8; j < n && j < w * 8 + 8; ++j) {
    const P* src = points + members[j] * f;
    P* dst = sorted + j * f;
    for (int k = lane; k < f; k += 32) dst[k] = src[k];
  }
}

constexpr int kMeanStages = 4;
constexpr int kMeanStageBytes = 24 * 1024;

// Centroid sums in member order from the member-ordered rows: one CTA per
// cluster streams its contiguous row range through a 4-stage ring of 1-D bulk
// copies; thread t owns factors t + 128 h and adds the rows strictly in order
// (numpy's mean(axis=0) adds rows one after another), then one divide.
template <class P>
__global__ void __launch_bounds__(128) centroid_stream_kernel(const P* __restrict__ sorted, int f,
                                                              const int64_t* __restrict__ offsets, int rows_per_stage,
                                                              int stage_bytes, double* __restrict__ centers) {
  extern __shared__ __align__(128) unsigned char mraw[];
  __shared__ __align__(8) uint64_t bars[kMeanStages];
  const int cl = blockIdx.x, t = threadIdx.x;
  const int64_t b = offsets[cl], e = offsets[cl + 1];
  if (e == b) return;
  const size_t rb = (size_t)f * sizeof(P);
  const int64_t nst = (e - b + rows_per_stage - 1) / rows_per_stage;
  const unsigned char* g = reinterpret_cast<const unsigned char*>(sorted);
  auto stage_range = [&](int64_t i, size_t& a0, uint32_t& sz, int& rows) {
    const int64_t r0 = b + i * rows_per_stage;
    const int64_t r1 = (r0 + rows_per_stage) < e ? (r0 + rows_per_stage) : e;
    rows = (int)(r1 - r0);
    a0 = ((size_t)r0 * rb) & ~size_t(15);
    sz = (uint32_t)((((size_t)r1 * rb) - a0 + 15) & ~size_t(15));
  };
  if (t == 0) {
    for (int q = 0; q < kMeanStages; ++q) sm100::mbar_init(bars + q, 1);
    sm100::fence_barrier_init();
  }
  __syncthreads();
  auto issue = [&](int64_t i) {
    size_t a0;
    uint32_t sz;
    int rows;
    stage_range(i, a0, sz, rows);
    const int q = (int)(i % kMeanStages);
    sm100::mbar_arrive_expect_tx(bars + q, sz);
    sm100::bulk_load_1d(mraw + (size_t)q * stage_bytes, g + a0, sz, bars + q);
  };
  if (t == 0)
    for (int64_t i = 0; i < nst && i < kMeanStages; ++i) issue(i);
  double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t i = 0; i < nst; ++i) {
    const int q = (int)(i % kMeanStages);
    sm100::mbar_wait(bars + q, (uint32_t)((i / kMeanStages) & 1));
    size_t a0;
    uint32_t sz;
    int rows;
    stage_range(i, a0, sz, rows);
    const P* x = reinterpret_cast<const P*>(mraw + (size_t)q * stage_bytes + (((size_t)(b + i * rows_per_stage) * rb) - a0));
#pragma unroll
    for (int h = 0; h < 8; ++h) {
      const int k = t + 128 * h;
      if (k < f) {
#pragma unroll 8
        for (int r = 0; r < rows; ++r) acc[h] += (double)x[(size_t)r * f + k];
      }
    }
    __syncthreads();  // stage q consumed by every thread
    if (t == 0 && i + kMeanStages < nst) {
      sm100::fence_proxy_async_smem();
      issue(i + kMeanStages);
    }
  }
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    const int k = t + 128 * h;
    if (k < f) centers[(int64_t)cl * f + k] = acc[h] / (double)(e - b);
  }
}

// centroid = (sum of the S part sums, in part order) / count; empty clusters
// keep their centroid (clustering.py:170-172)
__global__ void combine_mean_kernel(const double* __restrict__ psum, const int64_t* __restrict__ offsets, int c,
                                    int S, int f, double* __restrict__ centers) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)c * f) return;
  const int cl = (int)(i / f), k = (int)(i % f);
  const int64_t cnt = offsets[cl + 1] - offsets[cl];
  if (cnt == 0) return;
  double t = 0.0;
  for (int sp = 0; sp < S; ++sp) t += psum[((int64_t)cl * S + sp) * f + k];
  centers[i] = t / (double)cnt;
}

// Stable counting sort of points by cluster (members in (cluster, id)
// order): per-block cluster histograms, cluster totals + offsets, per
// (cluster, block) bases, then an in-order scatter per block.
constexpr int kGroupBlock = 1024;  // points per histogram / scatter block

__global__ void group_hist_kernel(const int64_t* __restrict__ assign, int64_t n, int c, int64_t nb,
                                  int32_t* __restrict__ bcount) {
  extern __shared__ int32_t h[];
  for (int i = threadIdx.x; i < c; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int64_t b0 = (int64_t)blockIdx.x * kGroupBlock;
  for (int64_t i = b0 + threadIdx.x; i < n && i < b0 + kGroupBlock; i += blockDim.x) atomicAdd(h + assign[i], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < c; i += blockDim.x) bcount[(int64_t)i * nb + blockIdx.x] = h[i];
}

// one warp per cluster: exclusive scan of its block counts in block order
__global__ void group_cluster_scan_kernel(int32_t* __restrict__ bcount, int64_t nb, int c,
                                          int64_t* __restrict__ totals) {
  const int cl = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (cl >= c) return;
  int32_t* row = bcount + (int64_t)cl * nb;
  int64_t carry = 0;
  for (int64_t b0 = 0; b0 < nb; b0 += 32) {
    const int64_t b = b0 + lane;
    const int64_t v = b < nb ? row[b] : 0;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (b < nb) row[b] = (int32_t)(carry + x - v);
    carry += __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) totals[cl] = carry;
}

__global__ void group_offsets_kernel(const int64_t* __restrict__ totals, int c, int64_t* __restrict__ out_counts,
                                     int64_t* __restrict__ offsets) {
  __shared__ int64_t wsum[32];
  __shared__ int64_t carry;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < c; c0 += blockDim.x) {
    const int i = c0 + t;
    const int64_t v = i < c ? totals[i] : 0;
    int64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int64_t pre = carry;
    for (int q = 0; q < w; ++q) pre += wsum[q];
    if (i < c) {
      offsets[i] = pre + x - v;
      out_counts[i] = v;
    }
    __syncthreads();
    if (t == 0)
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) carry += wsum[q];
    __syncthreads();
  }
  if (t == 0) offsets[c] = carry;
}

// one warp per block of points, in point order: ranks among equal clusters
// by match_any, a running per-cluster cursor in shared memory
__global__ void group_scatter_kernel(const int64_t* __restrict__ assign, int64_t n, int c, int64_t nb,
                                     const int32_t* __restrict__ bbase, const int64_t* __restrict__ offsets,
                                     int64_t* __restrict__ members) {
  extern __shared__ int32_t cur[];
  const int lane = threadIdx.x;
  const int64_t b = blockIdx.x;
  for (int i = lane; i < c; i += 32) cur[i] = 0;
  __syncwarp();
  const int64_t b0 = b * kGroupBlock;
  for (int64_t i0 = b0; i0 < n && i0 < b0 + kGroupBlock; i0 += 32) {
    const int64_t i = i0 + lane;
    const bool live = i < n && i < b0 + kGroupBlock;
    const int cl = live ? (int)assign[i] : -1;
    const unsigned live_m = __ballot_sync(0xffffffffu, live);
    const unsigned peers = __match_any_sync(0xffffffffu, cl) & live_m;
    const int leader = __ffs(peers) - 1;
    int base = 0;
    if (live && lane == leader) base = cur[cl];
    base = __shfl_sync(0xffffffffu, base, live ? leader : lane);
    if (live) {
      const int rank = __popc(peers & ((1u << lane) - 1u));
      members[offsets[cl] + bbase[(int64_t)cl * nb + b] + base + rank] = i;
    }
    __syncwarp();
    if (live && lane == leader) cur[cl] = base + __popc(peers);
    __syncwarp();
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

// ---------------------------------------------------------------------------
// persistent k-means++ seeding: one cooperative launch runs every pass.
// Per pass: (U) the D^2 update over 256-point chunks (as seed_update_kernel),
// grid barrier, (P) every CTA locates the next seed redundantly from the
// chunk sums (identical arithmetic in every CTA, so identical picks), CTA 0
// records it, all CTAs split the new seed's distances to the earlier seeds,
// grid barrier.  No launch or host round trip between passes.
// ---------------------------------------------------------------------------
struct SeedArgs {
  int64_t n;
  int f, k;
  const double* p2;
  const double* uniforms;
  int64_t* rows;
  double* centers;
  double* d2;
  int32_t* near;
  double* seed_c2;
  double* cd2;
  double* chunk_sums;
  double* range_sums;  // per CTA: sum of its contiguous chunk range
  int64_t nchunks;
  int32_t* degenerate;
  unsigned* barrier;
  unsigned long long* dbg;  // optional phase timers (ns): update, barrier 1, pick, barrier 2
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// all CTAs of the (co-resident) grid; `gen` counts barriers passed
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  ++gen;
  if (threadIdx.x == 0) {
    __threadfence();
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(bar), "r"(1u) : "memory");
    const unsigned want = gen * gridDim.x;
    while (ld_acquire_u32(bar) < want) __nanosleep(32);
    __threadfence();
  }
  __syncthreads();
}


// dynamic shared layout of seed_persistent_kernel: new-seed center, cached
// seed-seed distances and seed norms, per-warp double-buffered row staging
struct PSeedSmem {
  int kc;  // cached seeds (0: read cd2 / seed_c2 from global)
  size_t buf, cen_off, cdc_off, scc_off, bar_off, buf_off, total;
};

__host__ __device__ inline PSeedSmem pseed_smem(int f, size_t esize, int k, int wpb) {
  PSeedSmem m;
  const size_t row = (size_t)f * esize;
  m.buf = ((32 * row + 32) + 127) & ~size_t(127);
  m.kc = k <= 2048 ? k : 0;
  m.cen_off = 0;
  m.cdc_off = ((size_t)f * 8 + 15) & ~size_t(15);
  m.scc_off = m.cdc_off + (size_t)m.kc * 8;
  m.bar_off = (m.scc_off + (size_t)m.kc * 8 + 15) & ~size_t(15);
  m.buf_off = (m.bar_off + (size_t)wpb * 2 * 8 + 127) & ~size_t(127);
  m.total = m.buf_off + (size_t)wpb * 2 * m.buf;
  return m;
}

// inclusive scan of one double per thread over the CTA (warp shuffles +
// warp totals in fixed order); *total = the CTA sum
__device__ __forceinline__ double cta_scan(double x, double* wsum, double* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  double pre = 0.0, tot = 0.0;
  for (int q = 0; q < nw; ++q) {
    if (q < w) pre += wsum[q];
    tot += wsum[q];
  }
  *total = tot;
  return pre + x;
}

// First index i in [0, m) whose cumulative sum base + v[0] + ... + v[i]
// exceeds the target (numpy's searchsorted(cumsum, target, 'right')), scanned
// by the whole CTA: contiguous per-thread runs (held in registers when a run
// is at most 8 long, so every value is loaded once), a CTA scan, and the
// crossing run walked by its owner.  scale: the target is target * (total of
// v), so the top level scales its uniform by the total it has just summed.
// If rounding puts the target beyond the total, the last positive entry is
// taken.  Returns the index, the sum before it in *before and the total in
// *total (every thread gets the same values).  sh: 8 + 2 doubles of scratch.
template <class Get>
__device__ int64_t cta_crossing(Get get, int64_t m, double base, double target, bool scale, double* before,
                                double* total, double* sh) {
  const int t = threadIdx.x, CS = blockDim.x;
  double* wsum = sh;
  double* s_val = sh + 8;
  int64_t* s_idx = reinterpret_cast<int64_t*>(sh + 9);
  const int64_t per = (m + CS - 1) / CS;
  const int64_t c0 = t * per < m ? t * per : m, c1 = (c0 + per) < m ? (c0 + per) : m;
  const bool cached = per <= 8;
  double vv[8];
  double mine = 0.0;
  if (cached) {
#pragma unroll
    for (int i = 0; i < 8; ++i) vv[i] = c0 + i < c1 ? get(c0 + i) : 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) mine += vv[i];
  } else {
    for (int64_t b = c0; b < c1; b += 8) {
      double uu[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) uu[i] = b + i < c1 ? get(b + i) : 0.0;
#pragma unroll
      for (int i = 0; i < 8; ++i) mine += uu[i];
    }
  }
  if (t == 0) *s_idx = -1;
  const double incl = base + cta_scan(mine, wsum, total);  // its barrier orders the s_idx reset
  if (scale) target *= *total;
  const double excl = incl - mine;
  if (c0 < c1 && incl > target && !(excl > target)) {
    double acc = excl;
    int64_t c = c1;
    if (cached) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (c == c1 && c0 + i < c1) {
          if (vv[i] > 0.0 && acc + vv[i] > target)
            c = c0 + i;
          else
            acc += vv[i];
        }
    } else {
      for (int64_t q = c0; q < c1; ++q) {
        const double v = get(q);
        if (v > 0.0 && acc + v > target) {
          c = q;
          break;
        }
        acc += v;
      }
    }
    if (c == c1) {  // rounding between the summation orders: last positive entry of the run
      c = c1 - 1;
      while (c > c0 && !(get(c) > 0.0)) --c;
      acc = excl;
      for (int64_t q = c0; q < c; ++q) acc += get(q);
    }
    *s_idx = c;
    *s_val = acc;
  }
  __syncthreads();
  if (*s_idx < 0) {
    if (t == 0) {
      // rounding put the target outside this level's sums: beyond the total ->
      // last positive entry; before the base -> first positive entry
      int64_t c;
      if (target < base) {
        c = 0;
        while (c + 1 < m && !(get(c) > 0.0)) ++c;
      } else {
        c = m - 1;
        while (c > 0 && !(get(c) > 0.0)) --c;
      }
      double acc = base;
      for (int64_t q = 0; q < c; ++q) acc += get(q);
      *s_idx = c;
      *s_val = acc;
    }
    __syncthreads();
  }
  const int64_t r = *s_idx;
  *before = *s_val;
  __syncthreads();  // sh is reused by the next search
  return r;
}

template <class P>
__global__ void __launch_bounds__(256, 2) seed_persistent_kernel(const P* __restrict__ points, const SeedArgs a) {
  extern __shared__ __align__(128) unsigned char sm_raw[];
  __shared__ double pick_sh[10];
  const int f = a.f;
  const int64_t n = a.n;
  const int CS = blockDim.x, wpb = CS >> 5;  // chunk = one point per thread
  const PSeedSmem L = pseed_smem(f, sizeof(P), a.k, wpb);
  double* cen = reinterpret_cast<double*>(sm_raw + L.cen_off);
  double* cdc = reinterpret_cast<double*>(sm_raw + L.cdc_off);
  double* scc = reinterpret_cast<double*>(sm_raw + L.scc_off);
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm_raw + L.bar_off);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (lane == 0) {
    sm100::mbar_init(bars + 2 * w, 1);
    sm100::mbar_init(bars + 2 * w + 1, 1);
    sm100::fence_barrier_init();
  }
  const size_t row_bytes = (size_t)f * sizeof(P);
  const size_t total_bytes = (size_t)n * row_bytes;
  const unsigned char* gbase = reinterpret_cast<const unsigned char*>(points);
  const int64_t G = gridDim.x;
  uint32_t phbits = 0;  // mbarrier phase per staging buffer
  unsigned gen = 0;
  for (int q = t; q < f; q += CS) cen[q] = __ldcg(a.centers + q);
  __syncthreads();
  unsigned long long tm0 = 0, tm1 = 0, wait1 = 0;
  const bool timing = a.dbg && blockIdx.x == 0 && t == 0;
  const int64_t g0 = a.nchunks * blockIdx.x / G, g1 = a.nchunks * (blockIdx.x + 1) / G;
  const int64_t GW = wpb, r0 = g0 + w, r1 = g1;  // this CTA's contiguous range, warps interleaved
  for (int j = 0; j + 1 < a.k; ++j) {
    if (timing) tm0 = gtimer();
    const double u = a.uniforms[j];  // read here, used by the pick
    if (L.kc)
      for (int q = t; q <= j; q += CS) {
        scc[q] = __ldcg(a.seed_c2 + q);
        if (q < j) cdc[q] = __ldcg(a.cd2 + q);
      }
    __syncthreads();
    const double cc = L.kc ? scc[j] : __ldcg(a.seed_c2 + j);
    // 32-point slices: each CTA owns a contiguous range, its warps take the
    // slices round-robin and run their own pipelines (no CTA-wide step until
    // the range is done); the CTA then adds its range's slice sums in order
    // odd passes walk the range backwards: the slices read last are read
    // first again while they are still in L2
    const bool rev = j & 1;
    auto sl = [&](int64_t ch) { return rev ? g1 - 1 - (ch - g0) : ch; };
    // ------------------------------------------------------------ (U) update
    // per warp, a three-stage pipeline over this CTA's chunks: the test inputs
    // of chunk C load while chunk B's rows stream into one staging buffer and
    // chunk A (other buffer) is scored
    auto load_regs = [&](int64_t ch, double& mp2, double& old, int& an) {
      const int64_t me = sl(ch) * 32 + lane;
      mp2 = 0.0;
      old = DBL_MAX;
      an = 0;
      if (ch < r1 && me < n) {
        mp2 = a.p2[me];
        if (j > 0) {
          old = __ldcg(a.d2 + me);
          an = __ldcg(a.near + me);
        }
      }
    };
    auto test = [&](int64_t ch, double mp2, double old, int an) -> bool {
      if (ch >= r1) return false;
      const int64_t me = sl(ch) * 32 + lane;
      if (me >= n) return false;
      if (j == 0) return true;
      const double c2a = L.kc ? scc[an] : __ldcg(a.seed_c2 + an);
      const double cda = L.kc ? cdc[an] : __ldcg(a.cd2 + an);
      const double eta = 0x1p-40 * (mp2 + cc + c2a);
      return !(cda >= 4.0 * (old + eta) * (1.0 + 0x1p-30));
    };
    // stage the warp's 32 rows with one bulk copy when any of them is needed
    // (per-row copies of only the needed rows, by TMA or cp.async, measured
    // slower: issue rate); returns false when the rows are read from global
    auto issue = [&](int64_t ch, unsigned mask, int bsel) -> bool {
      if (!mask) return false;
      const int64_t u0 = sl(ch) * 32;
      const int64_t u1 = (u0 + 32) < n ? (u0 + 32) : n;
      const size_t start = (size_t)u0 * row_bytes, a0 = start & ~size_t(15);
      const size_t sz = ((size_t)u1 * row_bytes - a0 + 15) & ~size_t(15);
      if (a0 + sz > total_bytes) return false;  // buffer tail: read from global
      const unsigned char* src = gbase + a0;
      __syncwarp();
      if (lane == 0) {
        sm100::fence_proxy_async_smem();
        sm100::mbar_arrive_expect_tx(bars + 2 * w + bsel, (uint32_t)sz);
        sm100::bulk_load_1d(sm_raw + L.buf_off + (size_t)(2 * w + bsel) * L.buf, src, (uint32_t)sz,
                            bars + 2 * w + bsel);
      }
      return true;
    };
    int64_t chA = r0;
    double mp2A, oldA, mp2B, oldB;
    int anA, anB;
    load_regs(chA, mp2A, oldA, anA);
    bool needA = test(chA, mp2A, oldA, anA);
    unsigned mA = __ballot_sync(0xffffffffu, needA);
    int bA = 0;
    bool sA = issue(chA, mA, bA);
    int64_t chB = chA + GW;
    load_regs(chB, mp2B, oldB, anB);
    while (chA < r1) {
      const int64_t chC = chB + GW;
      const bool needB = test(chB, mp2B, oldB, anB);
      const unsigned mB = __ballot_sync(0xffffffffu, needB);
      const bool sB = issue(chB, mB, bA ^ 1);
      double mp2C, oldC;
      int anC;
      load_regs(chC, mp2C, oldC, anC);
      // score chunk A
      const int64_t slA = chA < r1 ? sl(chA) : chA;
      const int64_t meA = slA * 32 + lane;
      double fin = oldA;
      if (mA) {
        if (sA) {
          sm100::mbar_wait(bars + 2 * w + bA, (phbits >> bA) & 1u);
          phbits ^= 1u << bA;
        }
        if (needA) {  // scored in factor order: a duplicate of a seed gets exactly D^2 = 0
          double dot = 0.0;
          if (sA) {  // staged rows (shared-memory loads)
            const size_t s0 = (size_t)(slA * 32) * row_bytes;  // slice start
            const P* x = reinterpret_cast<const P*>(sm_raw + L.buf_off + (size_t)(2 * w + bA) * L.buf + (s0 & 15) +
                                                    (size_t)lane * row_bytes);
#pragma unroll 10
            for (int q = 0; q < f; ++q) dot = fma((double)x[q], cen[q], dot);
          } else {
            const P* x = points + meA * f;
#pragma unroll 5
            for (int q = 0; q < f; ++q) dot = fma((double)x[q], cen[q], dot);
          }
          double d = (mp2A + cc) - 2.0 * dot;
          d = d > 0.0 ? d : 0.0;
          if (j == 0 || d < oldA) {
            a.d2[meA] = d;
            a.near[meA] = j;
            fin = d;
          }
        }
      }
      double v = meA < n ? fin : 0.0;
      v = warp_sum(v);
      if (lane == 0) a.chunk_sums[slA] = v;
      chA = chB;
      mp2A = mp2B;
      oldA = oldB;
      needA = needB;
      mA = mB;
      sA = sB;
      bA ^= 1;
      chB = chC;
      mp2B = mp2C;
      oldB = oldC;
      anB = anC;
    }
    if (timing) {
      tm1 = gtimer();
      a.dbg[0] += tm1 - tm0;
      tm0 = tm1;
    }
    __syncthreads();
    if (t == 0) {  // this CTA's range of slice sums, in slice order
      double rs = 0.0;
      for (int64_t b = g0; b < g1; b += 8) {
        double vv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) vv[i] = b + i < g1 ? __ldcg(a.chunk_sums + b + i) : 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) rs += vv[i];
      }
      a.range_sums[blockIdx.x] = rs;
    }
    {
      unsigned long long tw0 = (a.dbg && t == 0) ? gtimer() : 0;
      grid_barrier(a.barrier, gen);
      if (a.dbg && t == 0) wait1 += gtimer() - tw0;
    }
    if (timing) {
      tm1 = gtimer();
      a.dbg[1] += tm1 - tm0;
      tm0 = tm1;
    }
    // ---------------------------------------------------------- (P) pick seed j+1
    // every CTA locates it with the same arithmetic (so the same pick): the
    // CTA range whose running sum crosses u * total, the slice inside that
    // range, the point inside that slice
    int64_t pp;
    {
      double before, total, sub;
      const int64_t rg = cta_crossing([&](int64_t q) { return __ldcg(a.range_sums + q); }, G, 0.0, u, true,
                                      &before, &total, pick_sh);
      if (!(total > 0.0)) {  // degenerate: every remaining pass takes the host branch
        if (blockIdx.x == 0 && t == 0) *a.degenerate = j + 1;
        break;
      }
      const double target = u * total;
      const int64_t x0 = a.nchunks * rg / G, x1 = a.nchunks * (rg + 1) / G;
      const int64_t chk = x0 + cta_crossing([&](int64_t q) { return __ldcg(a.chunk_sums + x0 + q); }, x1 - x0,
                                            before, target, false, &before, &sub, pick_sh);
      const int64_t pb = chk * 32, pe = (pb + 32) < n ? (pb + 32) : n;
      pp = pb + cta_crossing([&](int64_t q) { return __ldcg(a.d2 + pb + q); }, pe - pb, before, target, false,
                             &before, &sub, pick_sh);
    }
    const int64_t p = pp;
    for (int q = t; q < f; q += CS) {
      const double cv = (double)points[p * f + q];
      cen[q] = cv;
      if (blockIdx.x == 0) a.centers[(int64_t)(j + 1) * f + q] = cv;
    }
    if (blockIdx.x == 0 && t == 0) {
      a.rows[j + 1] = p;
      a.seed_c2[j + 1] = a.p2[p];
    }
    __syncthreads();
    // squared distances new seed -> seeds 0..j, one warp per seed across the grid
    for (int64_t q = (int64_t)blockIdx.x * wpb + w; q <= j; q += G * wpb) {
      const double* cq = a.centers + q * f;
      double acc = 0.0;
      for (int r = lane; r < f; r += 32) {
        const double d = cen[r] - __ldcg(cq + r);
        acc = fma(d, d, acc);
      }
      acc = warp_sum(acc);
      if (lane == 0) a.cd2[q] = acc;
    }
    if (timing) {
      tm1 = gtimer();
      a.dbg[2] += tm1 - tm0;
      tm0 = tm1;
    }
    grid_barrier(a.barrier, gen);
    if (timing) a.dbg[3] += gtimer() - tm0;
  }
  if (a.dbg && t == 0) {
    atomicAdd(a.dbg + 4, wait1);
    atomicMin(a.dbg + 5, wait1);
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
int fill_sqnorm(const void* px, int64_t n, int f, double* out, cudaStream_t s) {
  sqnorm_kernel<P><<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(static_cast<const P*>(px), n, f, out);
  SIMDEX_LAUNCH_CHECK("sqnorm");
  return SIMDEX_OK;
}

template <class P>
int assign_impl(const double* points, const float* points32, const P* px, int64_t n, int32_t f,
                const double* centers, int32_t c, const int64_t* prev, int64_t* out_assign, double* out_d2,
                int64_t* out_changed, double* out_objective, cudaStream_t s) {
  Scratch<double> p2, c2, part;
  SIMDEX_CUDA(c2.alloc(c, s));
  const bool tc = f + 1 <= kAssignGemmMaxF;  // (the tensor-core path keeps the squared norms in its workspace)
  if (!tc) {
    SIMDEX_CUDA(p2.alloc(n, s));
    if (int rc = fill_sqnorm<P>(px, n, f, p2.p, s)) return rc;
  }
  sqnorm_kernel<double><<<(unsigned)ceil_div(c, 256), 256, 0, s>>>(centers, c, f, c2.p);
  SIMDEX_LAUNCH_CHECK("sqnorm");
  SIMDEX_CUDA(cudaMemsetAsync(out_changed, 0, sizeof(int64_t), s));
  auto* changed = reinterpret_cast<unsigned long long*>(out_changed);
  if (tc) {
    // tensor-core candidates + exact float64 d2; overflowing bands go to the SIMT kernel
    Scratch<int64_t> over;
    Scratch<int32_t> n_over;
    SIMDEX_CUDA(over.alloc(n, s));
    SIMDEX_CUDA(n_over.alloc(1, s));
    const double* p2w = nullptr;  // in the context workspace: valid until the context's next call
    int rc = gemm_kmeans_assign(points, points32, n, f, &fill_sqnorm<P>, &p2w, centers, c2.p, c, prev, out_assign,
                                out_d2, changed, over.p, n_over.p, s);
    if (rc) return rc;
    // rows whose band overflowed (rare): exact SIMT kernel, count read on the device
    assign_kernel<P><<<(unsigned)std::min<int64_t>(ceil_div(n, kAssignThreads), 2 * sm_count()), kAssignThreads, 0,
                       s>>>(px, p2w, n, f, centers, c2.p, c, prev, out_assign, out_d2, changed, over.p, n_over.p);
    SIMDEX_LAUNCH_CHECK("assign");
  } else {
    ProfileScope _prof("kmeans_assign", s);
    assign_kernel<P><<<(unsigned)ceil_div(n, kAssignThreads), kAssignThreads, 0, s>>>(
        px, p2.p, n, f, centers, c2.p, c, prev, out_assign, out_d2, changed, nullptr, nullptr);
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
  if (k == 1) return SIMDEX_OK;
  {
    // one cooperative launch for every pass (grid = co-resident CTAs, two per
    // SM); the chunk is one point per thread, 32 per warp
    // CTA size by resident warps per SM (staging buffers bound them)
    int wpb = 0, occ = 0;
    size_t psm = 0;
    for (int cand = 8; cand >= 1; cand >>= 1) {
      const size_t sm_c = pseed_smem(f, sizeof(P), k, cand).total;
      if (sm_c > 200 * 1024) continue;
      SIMDEX_CUDA(cudaFuncSetAttribute(seed_persistent_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)sm_c));
      int o = 0;
      SIMDEX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, seed_persistent_kernel<P>, 32 * cand, sm_c));
      if (o * cand > occ * wpb) {
        wpb = cand;
        occ = o;
        psm = sm_c;
      }
    }
    if (occ >= 1) {
      SIMDEX_CUDA(cudaFuncSetAttribute(seed_persistent_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)psm));
      const int64_t cs = 32 * wpb, nch = ceil_div(n, 32);  // 32-point slices
      Scratch<unsigned> bar;
      Scratch<double> csum, rsum;
      int64_t grid = (int64_t)occ * sm_count();
      if (grid > nch) grid = nch;
      SIMDEX_CUDA(bar.alloc(1, s));
      SIMDEX_CUDA(csum.alloc(nch, s));
      SIMDEX_CUDA(rsum.alloc(grid, s));
      SIMDEX_CUDA(cudaMemsetAsync(bar.p, 0, sizeof(unsigned), s));
      SeedArgs a{};
      a.n = n;
      a.f = f;
      a.k = k;
      a.p2 = p2.p;
      a.uniforms = uniforms;
      a.rows = out_rows;
      a.centers = out_centers;
      a.d2 = d2.p;
      a.near = near.p;
      a.seed_c2 = seed_c2.p;
      a.cd2 = cd2.p;
      a.chunk_sums = csum.p;
      a.range_sums = rsum.p;
      a.nchunks = nch;
      a.degenerate = out_deg;
      a.barrier = bar.p;
      Scratch<unsigned long long> dbg;
      const bool timing = std::getenv("SIMDEX_SEED_TIMING") != nullptr;
      if (timing) {
        SIMDEX_CUDA(dbg.alloc(6, s));
        SIMDEX_CUDA(cudaMemsetAsync(dbg.p, 0, 5 * sizeof(unsigned long long), s));
        SIMDEX_CUDA(cudaMemsetAsync(dbg.p + 5, 0xff, sizeof(unsigned long long), s));
        a.dbg = dbg.p;
      }
      const P* pts = points;
      void* args[] = {(void*)&pts, (void*)&a};
      ProfileScope _prof("seed_persistent", s);
      SIMDEX_CUDA(cudaLaunchCooperativeKernel((const void*)seed_persistent_kernel<P>, dim3((unsigned)grid),
                                              dim3((unsigned)cs), args, psm, s));
      _prof.end();
      count_launches(1);
      if (timing) {
        unsigned long long h[6];
        SIMDEX_CUDA(cudaMemcpyAsync(h, dbg.p, sizeof(h), cudaMemcpyDeviceToHost, s));
        SIMDEX_CUDA(cudaStreamSynchronize(s));
        fprintf(stderr,
                "[simdex] seed grid %lld x %lld: update %.3f ms barrier %.3f ms pick %.3f ms barrier %.3f ms; "
                "barrier-1 wait per CTA: mean %.1f us min %.1f us (%lld points)\n",
                (long long)grid, (long long)cs, h[0] * 1e-6, h[1] * 1e-6, h[2] * 1e-6, h[3] * 1e-6,
                (double)h[4] / grid * 1e-3, (double)h[5] * 1e-3, (long long)n);
      }
      return SIMDEX_OK;
    }
  }
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
int mean_impl(const P* points, int64_t n, int32_t f, const int64_t* members, const int64_t* offsets, int32_t c,
              double* centers, cudaStream_t s) {
  if (f > kSeqMaxF) {
    set_error("kmeans_update: f > %d unsupported", kSeqMaxF);
    return SIMDEX_EUNSUPPORTED;
  }
  const size_t rb = (size_t)f * sizeof(P);
  if (rb + 32 <= (size_t)kMeanStageBytes) {
    // member-ordered copy, then contiguous streamed sums
    Scratch<P> sorted;
    SIMDEX_CUDA(sorted.alloc((size_t)n * f + 64 / sizeof(P), s));  // + slack for 16-byte rounded copies
    gather_rows_kernel<P><<<(unsigned)ceil_div(n, 64), 256, 0, s>>>(points, f, members, n, sorted.p);
    SIMDEX_LAUNCH_CHECK("gather_rows");
    const int rows = (int)((kMeanStageBytes - 32) / rb);
    const size_t smem = (size_t)kMeanStages * kMeanStageBytes;
    SIMDEX_CUDA(cudaFuncSetAttribute(centroid_stream_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    ProfileScope _prof("centroid_mean", s);
    centroid_stream_kernel<P><<<(unsigned)c, 128, smem, s>>>(sorted.p, f, offsets, rows, kMeanStageBytes, centers);
    _prof.end();
    SIMDEX_LAUNCH_CHECK("centroid_mean");
    return SIMDEX_OK;
  }
  // wide rows: gather-staged kernel
  int rows = (int)((110 * 1024) / (2 * rb));
  rows = rows > 256 ? 256 : (rows < 1 ? 1 : rows);
  const size_t smem = 2 * (size_t)rows * rb;
  SIMDEX_CUDA(cudaFuncSetAttribute(centroid_seq_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ProfileScope _prof("centroid_mean", s);
  centroid_seq_kernel<P><<<(unsigned)c, 128, smem, s>>>(points, f, members, offsets, rows, centers);
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

namespace simdex {
// counting sort for c <= 8192, the merge sort otherwise
cudaError_t group_stable(const int64_t* assign, int64_t n, int c, int64_t* out_counts, int64_t* out_members,
                         int64_t* out_offsets, cudaStream_t s) {
  if (c <= 8192) {
    const int64_t nb = ceil_div(n, kGroupBlock) > 0 ? ceil_div(n, kGroupBlock) : 1;
    Scratch<int32_t> bcount;
    Scratch<int64_t> totals;
    SIMDEX_TRY(bcount.alloc((size_t)c * nb, s));
    SIMDEX_TRY(totals.alloc(c, s));
    group_hist_kernel<<<(unsigned)nb, 256, sizeof(int32_t) * c, s>>>(assign, n, c, nb, bcount.p);
    group_cluster_scan_kernel<<<(unsigned)ceil_div(c, 8), 256, 0, s>>>(bcount.p, nb, c, totals.p);
    group_offsets_kernel<<<1, 1024, 0, s>>>(totals.p, c, out_counts, out_offsets);
    if (n > 0)
      group_scatter_kernel<<<(unsigned)nb, 32, sizeof(int32_t) * c, s>>>(assign, n, c, nb, bcount.p, out_offsets,
                                                                        out_members);
    count_launches(n > 0 ? 4 : 3);
    return cudaGetLastError();
  }
  Scratch<double> keys;
  Scratch<int32_t> ids;
  Scratch<unsigned long long> cnt;
  SIMDEX_TRY(keys.alloc(n, s));
  SIMDEX_TRY(ids.alloc(n, s));
  SIMDEX_TRY(cnt.alloc(c, s));
  cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * c, s);
  if (n > 0) {
    cluster_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(assign, n, keys.p, ids.p, cnt.p);
    cudaError_t e = segmented_sort_desc(keys.p, ids.p, 1, n, s);
    if (e != cudaSuccess) return e;
  }
  offsets_kernel<<<1, 32, 0, s>>>(cnt.p, c, out_counts, out_offsets);
  if (n > 0) members_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(ids.p, n, out_members);
  count_launches(n > 0 ? 3 : 1);
  return cudaGetLastError();
}
}  // namespace simdex

extern "C" int simdex_kmeans_update(const double* points, const float* points32, int64_t n, int32_t f,
                                    const int64_t* assign, int32_t c, double* centers, int64_t* out_counts,
                                    int64_t* out_members, int64_t* out_offsets, void* stream) {
  SIMDEX_CHECK_ARG((points || points32) && assign && out_counts && out_members && out_offsets,
                   "simdex_kmeans_update: null pointer");
  SIMDEX_CHECK_ARG(n >= 1 && f >= 1 && c >= 1 && n < INT32_MAX, "simdex_kmeans_update: bad sizes");
  cudaStream_t s = as_stream(stream);
  SIMDEX_CUDA(group_stable(assign, n, c, out_counts, out_members, out_offsets, s));
  if (!centers) return SIMDEX_OK;  // grouping only (members/offsets/counts)
  if (points32) return mean_impl<float>(points32, n, f, out_members, out_offsets, c, centers, s);
  return mean_impl<double>(points, n, f, out_members, out_offsets, c, centers, s);
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
