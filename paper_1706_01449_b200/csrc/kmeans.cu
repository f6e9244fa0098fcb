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

namespace simdex {
namespace {

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
    double* __restrict__ out_d2, unsigned long long* __restrict__ changed, double* __restrict__ block_sums) {
  __shared__ double cs[kCC][kFC + 1];
  __shared__ double red[kAssignThreads / 32];
  const int64_t u = (int64_t)blockIdx.x * kAssignThreads + threadIdx.x;
  const bool live = u < n;
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
    block_sums[blockIdx.x] = s;
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

// One CTA (256 threads) per cluster: thread (lane_m, k) sums members
// lane_m, lane_m + L, ... of factor k; the L partials are then added in lane
// order.  Fixed partition and order: deterministic.  Empty clusters keep
// their centroid (clustering.py:170-172).
template <class P>
__global__ void __launch_bounds__(256) centroid_mean_kernel(const P* __restrict__ points, int f,
                                                            const int64_t* __restrict__ members,
                                                            const int64_t* __restrict__ offsets,
                                                            double* __restrict__ centers) {
  __shared__ double part[256];
  const int c = blockIdx.x;
  const int64_t b = offsets[c], e = offsets[c + 1];
  if (e == b) return;
  const int L = f >= 256 ? 1 : 256 / f;
  for (int k0 = 0; k0 < f; k0 += 256) {
    const int fk = (f - k0) < 256 ? (f - k0) : 256;
    const int t = threadIdx.x;
    const int ml = f >= 256 ? 0 : t / fk, k = f >= 256 ? t : t % fk;
    double s = 0.0;
    if (ml < L && k < fk)
      for (int64_t m = b + ml; m < e; m += L) s += (double)points[members[m] * f + k0 + k];
    part[t] = s;
    __syncthreads();
    if (t < fk) {
      double tot = 0.0;
      for (int l = 0; l < L; ++l) tot += part[l * fk + t];
      centers[(int64_t)c * f + k0 + t] = tot / (double)(e - b);
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
template <class P>
__global__ void __launch_bounds__(kSeedThreads) seed_update_kernel(const P* __restrict__ points,
                                                                   const double* __restrict__ p2, int64_t n, int f,
                                                                   const int64_t* __restrict__ rows, int j,
                                                                   double* __restrict__ d2,
                                                                   double* __restrict__ block_sums,
                                                                   const int32_t* __restrict__ degenerate) {
  extern __shared__ double cen[];
  __shared__ double red[kSeedThreads / 32];
  if (*degenerate >= 0) return;
  const int64_t r = rows[j];
  for (int k = threadIdx.x; k < f; k += kSeedThreads) cen[k] = (double)points[r * f + k];
  __syncthreads();
  const double cc = p2[r];
  const int64_t u = (int64_t)blockIdx.x * kSeedThreads + threadIdx.x;
  double v = 0.0;
  if (u < n) {
    const P* x = points + u * f;
    double dot = 0.0;
    for (int k = 0; k < f; ++k) dot = fma((double)x[k], cen[k], dot);
    double d = (p2[u] + cc) - 2.0 * dot;
    d = d > 0.0 ? d : 0.0;
    v = (j == 0) ? d : fmin(d2[u], d);
    d2[u] = v;
  }
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kSeedThreads / 32; ++w) s += red[w];
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
  for (int k = t; k < f; k += blockDim.x) centers[(int64_t)(j + 1) * f + k] = (double)points[p * f + k];
}

template <class P>
__global__ void seed_first_kernel(const P* __restrict__ points, int f, int64_t first, int64_t* rows, double* centers,
                                  int32_t* degenerate) {
  if (threadIdx.x == 0) {
    rows[0] = first;
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
int assign_impl(const P* points, int64_t n, int32_t f, const double* centers, int32_t c, const int64_t* prev,
                int64_t* out_assign, double* out_d2, int64_t* out_changed, double* out_objective, cudaStream_t s) {
  Scratch<double> p2, c2, part;
  const int64_t nb = ceil_div(n, kAssignThreads);
  SIMDEX_CUDA(p2.alloc(n, s));
  SIMDEX_CUDA(c2.alloc(c, s));
  SIMDEX_CUDA(part.alloc(nb, s));
  sqnorm_kernel<P><<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(points, n, f, p2.p);
  SIMDEX_LAUNCH_CHECK("sqnorm");
  sqnorm_kernel<double><<<(unsigned)ceil_div(c, 256), 256, 0, s>>>(centers, c, f, c2.p);
  SIMDEX_LAUNCH_CHECK("sqnorm");
  SIMDEX_CUDA(cudaMemsetAsync(out_changed, 0, sizeof(int64_t), s));
  ProfileScope _prof("kmeans_assign", s);
  assign_kernel<P><<<(unsigned)nb, kAssignThreads, 0, s>>>(points, p2.p, n, f, centers, c2.p, c, prev, out_assign,
                                                           out_d2, reinterpret_cast<unsigned long long*>(out_changed),
                                                           part.p);
  _prof.end();
  SIMDEX_LAUNCH_CHECK("assign");
  sum_partials_kernel<<<1, 1024, 0, s>>>(part.p, nb, out_objective);
  SIMDEX_LAUNCH_CHECK("sum_partials");
  return SIMDEX_OK;
}

template <class P>
int seed_impl(const P* points, int64_t n, int32_t f, int32_t k, int64_t first, const double* uniforms,
              int64_t* out_rows, double* out_centers, int32_t* out_deg, cudaStream_t s) {
  const int64_t nb = ceil_div(n, kSeedThreads);
  Scratch<double> p2, d2, part;
  SIMDEX_CUDA(p2.alloc(n, s));
  SIMDEX_CUDA(d2.alloc(n, s));
  SIMDEX_CUDA(part.alloc(nb, s));
  sqnorm_kernel<P><<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(points, n, f, p2.p);
  SIMDEX_LAUNCH_CHECK("sqnorm");
  seed_first_kernel<P><<<1, 128, 0, s>>>(points, f, first, out_rows, out_centers, out_deg);
  SIMDEX_LAUNCH_CHECK("seed_first");
  const size_t smem = (size_t)f * sizeof(double);
  if (smem > 48 * 1024)
    SIMDEX_CUDA(cudaFuncSetAttribute(seed_update_kernel<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int j = 0; j + 1 < k; ++j) {
    ProfileScope _prof("seed_update", s);
    seed_update_kernel<P><<<(unsigned)nb, kSeedThreads, smem, s>>>(points, p2.p, n, f, out_rows, j, d2.p, part.p,
                                                                   out_deg);
    _prof.end();
    ProfileScope _prof2("seed_pick", s);
    seed_pick_kernel<P><<<1, kPickThreads, 0, s>>>(points, n, f, d2.p, part.p, nb, uniforms, j, out_rows, out_centers,
                                                   out_deg);
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
  centroid_mean_kernel<P><<<(unsigned)c, 256, 0, s>>>(points, f, members, offsets, centers);
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
    return assign_impl<float>(points32, n, f, centers, c, prev_assign, out_assign, out_d2, out_changed, out_objective,
                              s);
  return assign_impl<double>(points, n, f, centers, c, prev_assign, out_assign, out_d2, out_changed, out_objective, s);
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
