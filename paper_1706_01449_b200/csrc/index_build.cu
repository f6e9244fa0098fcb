// SimDex index construction on device (index.py:90-155, clustering.py:65-93):
//   * per-(cluster, item) half-angle theta_ic and Eq. 2 ceiling in float64,
//   * per-cluster theta_b (max member angle) via an order-free atomic max,
//   * a batched merge sort of every cluster's list by (ceiling desc, id asc):
//     2048-element tiles sorted in shared memory (8 per thread in registers,
//     then merge-path merges), then merge passes whose CTAs stage their two
//     input ranges in shared memory (keys are unique because ids are).
#include <cfloat>
#include <cmath>

#include "common.cuh"

namespace simdex {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortItems = 8;                           // elements per thread
constexpr int kSortTile = kSortThreads * kSortItems;  // elements per CTA tile

__device__ __forceinline__ bool kv_before(double ka, int32_t ia, double kb, int32_t ib) {
  // (key desc, id asc); -0.0 == +0.0 like numpy's comparisons
  return ka > kb || (ka == kb && ia < ib);
}

// Shared-memory slot of tile element e: one pad slot per 8 elements, so a
// thread's 8 consecutive elements (stride 8 across the warp) hit distinct banks.
__device__ __forceinline__ int pad8(int e) { return e + (e >> 3); }
constexpr int kSortSlots = kSortTile + kSortTile / 8;

// Number of A elements among the first d outputs of merge(A, B) (merge path);
// A(i) / B(j) return (key, id) of the i-th / j-th element.
template <class FA, class FB>
__device__ __forceinline__ int merge_split(FA A, int la, FB B, int lb, int d) {
  int lo = d - lb > 0 ? d - lb : 0, hi = d < la ? d : la;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    double ka, kb;
    int32_t ia, ib;
    A(mid, ka, ia);
    B(d - mid - 1, kb, ib);
    if (kv_before(ka, ia, kb, ib))
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// kSortItems outputs of merge(A, B) starting at (i, j), into registers
// (padding (-inf, INT32_MAX) once both inputs are exhausted)
template <class FA, class FB>
__device__ __forceinline__ void merge_run(FA A, int la, FB B, int lb, int i, int j, double* rk, int32_t* ri) {
  double ka = -DBL_MAX, kb = -DBL_MAX;
  int32_t ia = INT32_MAX, ib = INT32_MAX;
  if (i < la) A(i, ka, ia);
  if (j < lb) B(j, kb, ib);
#pragma unroll
  for (int t = 0; t < kSortItems; ++t) {
    const bool takeA = i < la && (j >= lb || kv_before(ka, ia, kb, ib));
    if (takeA) {
      rk[t] = ka;
      ri[t] = ia;
      if (++i < la) A(i, ka, ia);
    } else {
      rk[t] = j < lb ? kb : -DBL_MAX;
      ri[t] = j < lb ? ib : INT32_MAX;
      if (++j < lb) B(j, kb, ib);
    }
  }
}

// Sort every kSortTile-element tile of every segment: 8 elements per thread
// sorted in registers, then merge-path merges of doubling runs in shared memory.
__global__ void __launch_bounds__(kSortThreads) tile_sort_kernel(double* keys, int32_t* ids, int64_t len,
                                                                 int64_t tiles_per_seg) {
  __shared__ double sk[kSortSlots];
  __shared__ int32_t si[kSortSlots];
  const int64_t seg = blockIdx.x / tiles_per_seg, tile = blockIdx.x % tiles_per_seg;
  const int64_t base = seg * len + tile * kSortTile;
  const int n = (int)((len - tile * kSortTile) < kSortTile ? (len - tile * kSortTile) : kSortTile);
  const int t = threadIdx.x;
  for (int e = t; e < kSortTile; e += kSortThreads) {  // coalesced; padding sorts last
    sk[pad8(e)] = e < n ? keys[base + e] : -DBL_MAX;
    si[pad8(e)] = e < n ? ids[base + e] : INT32_MAX;
  }
  __syncthreads();
  double rk[kSortItems];
  int32_t ri[kSortItems];
#pragma unroll
  for (int q = 0; q < kSortItems; ++q) {
    rk[q] = sk[pad8(t * kSortItems + q)];
    ri[q] = si[pad8(t * kSortItems + q)];
  }
  // odd-even transposition network over the thread's 8 elements
#pragma unroll
  for (int r = 0; r < kSortItems; ++r) {
#pragma unroll
    for (int q = r & 1; q + 1 < kSortItems; q += 2) {
      if (kv_before(rk[q + 1], ri[q + 1], rk[q], ri[q])) {
        const double tk = rk[q];
        rk[q] = rk[q + 1];
        rk[q + 1] = tk;
        const int32_t ti = ri[q];
        ri[q] = ri[q + 1];
        ri[q + 1] = ti;
      }
    }
  }
  for (int w = kSortItems; w < kSortTile; w <<= 1) {
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kSortItems; ++q) {
      sk[pad8(t * kSortItems + q)] = rk[q];
      si[pad8(t * kSortItems + q)] = ri[q];
    }
    __syncthreads();
    const int o = t * kSortItems, a0 = (o / (2 * w)) * (2 * w), d = o - a0;
    auto A = [&](int i, double& k, int32_t& id) {
      k = sk[pad8(a0 + i)];
      id = si[pad8(a0 + i)];
    };
    auto B = [&](int j, double& k, int32_t& id) {
      k = sk[pad8(a0 + w + j)];
      id = si[pad8(a0 + w + j)];
    };
    const int i = merge_split(A, w, B, w, d);
    merge_run(A, w, B, w, i, d - i, rk, ri);
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < kSortItems; ++q) {
    sk[pad8(t * kSortItems + q)] = rk[q];
    si[pad8(t * kSortItems + q)] = ri[q];
  }
  __syncthreads();
  for (int e = t; e < n; e += kSortThreads) {
    keys[base + e] = sk[pad8(e)];
    ids[base + e] = si[pad8(e)];
  }
}

// Merge adjacent sorted runs of width w inside every segment, src -> dst; each
// CTA writes one kSortTile-element output tile (tiles never straddle a pair:
// 2w is a multiple of the tile).  Its A and B ranges are found by a merge-path
// search over global memory, staged in shared memory, and merged there.
__global__ void __launch_bounds__(kSortThreads) merge_pass_kernel(const double* __restrict__ sk,
                                                                  const int32_t* __restrict__ si, double* dk,
                                                                  int32_t* di, int64_t len, int64_t w,
                                                                  int64_t tiles_per_seg) {
  __shared__ double tk[kSortSlots];
  __shared__ int32_t ti[kSortSlots];
  __shared__ int s_split[2];
  const int64_t seg = blockIdx.x / tiles_per_seg, tile = blockIdx.x % tiles_per_seg;
  const int64_t o0 = tile * kSortTile;  // output offset within the segment
  const int n = (int)((len - o0) < kSortTile ? (len - o0) : kSortTile);
  const int64_t a0 = (o0 / (2 * w)) * (2 * w);
  const int64_t la64 = (len - a0) < w ? (len - a0) : w;
  const int64_t b0 = a0 + la64;
  const int64_t lb64 = (len - b0) < w ? ((len - b0) > 0 ? (len - b0) : 0) : w;
  const int la = (int)la64, lb = (int)lb64;
  const double* Ak = sk + seg * len + a0;
  const int32_t* Ai = si + seg * len + a0;
  const double* Bk = Ak + la;
  const int32_t* Bi = Ai + la;
  const int t = threadIdx.x;
  const int d0 = (int)(o0 - a0), d1 = d0 + n;
  auto GA = [&](int i, double& k, int32_t& id) {
    k = __ldg(Ak + i);
    id = __ldg(Ai + i);
  };
  auto GB = [&](int j, double& k, int32_t& id) {
    k = __ldg(Bk + j);
    id = __ldg(Bi + j);
  };
  if (t == 0) s_split[0] = merge_split(GA, la, GB, lb, d0);
  if (t == 32) s_split[1] = merge_split(GA, la, GB, lb, d1);
  __syncthreads();
  const int i0 = s_split[0], i1 = s_split[1];
  const int na = i1 - i0, j0 = d0 - i0, nb = n - na;
  for (int e = t; e < n; e += kSortThreads) {  // A part then B part, coalesced
    if (e < na) {
      tk[pad8(e)] = __ldg(Ak + i0 + e);
      ti[pad8(e)] = __ldg(Ai + i0 + e);
    } else {
      tk[pad8(e)] = __ldg(Bk + j0 + e - na);
      ti[pad8(e)] = __ldg(Bi + j0 + e - na);
    }
  }
  __syncthreads();
  double rk[kSortItems];
  int32_t ri[kSortItems];
  const int d = t * kSortItems;
  if (d < n) {
    auto A = [&](int i, double& k, int32_t& id) {
      k = tk[pad8(i)];
      id = ti[pad8(i)];
    };
    auto B = [&](int j, double& k, int32_t& id) {
      k = tk[pad8(na + j)];
      id = ti[pad8(na + j)];
    };
    const int i = merge_split(A, na, B, nb, d);
    merge_run(A, na, B, nb, i, d - i, rk, ri);
  }
  __syncthreads();
  if (d < n) {
#pragma unroll
    for (int q = 0; q < kSortItems; ++q) {
      tk[pad8(d + q)] = rk[q];  // positions past n hold padding and are not written out
      ti[pad8(d + q)] = ri[q];
    }
  }
  __syncthreads();
  double* D = dk + seg * len + o0;
  int32_t* Di = di + seg * len + o0;
  for (int e = t; e < n; e += kSortThreads) {
    D[e] = tk[pad8(e)];
    Di[e] = ti[pad8(e)];
  }
}

// ---------------------------------------------------------------------------
// ceilings (index.py:103-121)
// ---------------------------------------------------------------------------
__global__ void item_norms_kernel(const double* __restrict__ items, int64_t ni, int f, double* __restrict__ norms) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ni) return;
  const double* x = items + i * f;
  double s = 0.0;
  for (int k = 0; k < f; ++k) s = fma(x[k], x[k], s);
  norms[i] = sqrt(s);
}

// unit item directions x / |x| (the division index.py's angle takes per
// (cluster, item) pair, done once per item here), stored factor-major
// ([f][ni]) so a warp's 32 items read one coalesced line per factor; zero
// rows stay zero
__global__ void unit_cols_kernel(const double* __restrict__ items, const double* __restrict__ norms, int64_t ni, int f,
                                 double* __restrict__ unit) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ni * f) return;
  const int64_t i = e / f;
  const int k = (int)(e - i * f);
  const double nrm = norms[i];
  unit[(int64_t)k * ni + i] = nrm == 0.0 ? 0.0 : items[e] / nrm;
}

constexpr int kBoundGroup = 16;  // clusters per CTA: each item direction is read once per group

// grid: (ceil(ni/128), ceil(c/16)).  Thread = item; it accumulates the
// half-angle sums for 16 clusters at once (unit centroids in shared memory),
// then writes keys = ceiling, ids = item id for the sort.
__global__ void __launch_bounds__(128) bounds_kernel(const double* __restrict__ unit,
                                                     const double* __restrict__ norms, int64_t ni, int f, int c,
                                                     const double* __restrict__ centers,
                                                     const double* __restrict__ theta, double* __restrict__ keys,
                                                     int32_t* __restrict__ ids) {
  extern __shared__ double y[];  // [kBoundGroup][f] unit centroids
  __shared__ double s_cn[kBoundGroup];
  const int c0 = blockIdx.y * kBoundGroup;
  const int ng = (c - c0) < kBoundGroup ? (c - c0) : kBoundGroup;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int g = w; g < ng; g += blockDim.x >> 5) {  // centroid norms, one warp each
    const double* cen = centers + (int64_t)(c0 + g) * f;
    if (lane == 0) {
      double s = 0.0;
      for (int k = 0; k < f; ++k) s = fma(cen[k], cen[k], s);
      s_cn[g] = sqrt(s);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < ng * f; e += blockDim.x) {
    const int g = e / f;
    const double cn = s_cn[g];
    y[e] = cn > 0.0 ? centers[(int64_t)c0 * f + e] / cn : 0.0;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ni) return;
  double dm[kBoundGroup], dp[kBoundGroup];
#pragma unroll
  for (int g = 0; g < kBoundGroup; ++g) dm[g] = dp[g] = 0.0;
  for (int k = 0; k < f; ++k) {
    const double xk = __ldg(unit + (int64_t)k * ni + i);
#pragma unroll
    for (int g = 0; g < kBoundGroup; ++g) {
      const double yk = y[g * f + k];
      const double a = xk - yk, b = xk + yk;
      dm[g] = fma(a, a, dm[g]);
      dp[g] = fma(b, b, dp[g]);
    }
  }
  const double nrm = norms[i];
#pragma unroll
  for (int g = 0; g < kBoundGroup; ++g) {
    if (g < ng) {
      const double ang = (s_cn[g] == 0.0 || nrm == 0.0) ? M_PI / 2.0 : 2.0 * atan2(sqrt(dm[g]), sqrt(dp[g]));
      const double slack = theta[c0 + g];
      double bound = (slack < ang) ? nrm * cos(ang - slack) : nrm;
      if (bound == 0.0) bound = 0.0;  // fold -0.0
      keys[(int64_t)(c0 + g) * ni + i] = bound;
      ids[(int64_t)(c0 + g) * ni + i] = (int32_t)i;
    }
  }
}

// theta_b: per-user angle to its centroid, atomic max on the (non-negative) bits.
// unit_centers[c, k] = centers[c, k] / ||c|| is divided once per centre
// (unit_centers_kernel) instead of once per user: the same quotients.
__global__ void max_angles_kernel(const double* __restrict__ users, int64_t n, int f,
                                  const double* __restrict__ unit_centers, const double* __restrict__ cnorm,
                                  const int64_t* __restrict__ assign, unsigned long long* __restrict__ theta_bits) {
  int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t c = assign[u];
  const double* x = users + u * f;
  const double* y = unit_centers + c * f;
  const double cn = cnorm[c];
  double s = 0.0;
  for (int k = 0; k < f; ++k) s = fma(x[k], x[k], s);
  const double un = sqrt(s);
  double ang;
  if (cn == 0.0 || un == 0.0) {
    ang = M_PI;  // DEGENERATE_ANGLE (clustering.py:21-23)
  } else {
    double dm = 0.0, dp = 0.0;
    for (int k = 0; k < f; ++k) {
      double xk = x[k] / un, yk = y[k];
      double a = xk - yk, b = xk + yk;
      dm = fma(a, a, dm);
      dp = fma(b, b, dp);
    }
    ang = 2.0 * atan2(sqrt(dm), sqrt(dp));
  }
  atomicMax(theta_bits + c, (unsigned long long)__double_as_longlong(ang));
}

__global__ void unit_centers_kernel(const double* __restrict__ centers, const double* __restrict__ cnorm, int64_t c,
                                    int f, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= c * f) return;
  const double cn = cnorm[t / f];
  out[t] = cn == 0.0 ? 0.0 : centers[t] / cn;
}

// pos[c, list_ids[c, j]] = j  (inverse permutation of every cluster's list)
__global__ void list_pos_kernel(const int32_t* __restrict__ ids, int64_t c, int64_t n, int32_t* __restrict__ pos) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= c * n) return;
  const int64_t row = t / n;
  pos[row * n + ids[t]] = (int32_t)(t - row * n);
}

__global__ void center_norms_kernel(const double* __restrict__ centers, int c, int f, double* __restrict__ out) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= c) return;
  double s = 0.0;
  for (int k = 0; k < f; ++k) s = fma(centers[(int64_t)j * f + k], centers[(int64_t)j * f + k], s);
  out[j] = sqrt(s);
}

}  // namespace

cudaError_t segmented_sort_desc(double* keys, int32_t* ids, int64_t segs, int64_t len, cudaStream_t s) {
  if (segs == 0 || len <= 1) return cudaSuccess;
  const int64_t tiles = ceil_div(len, kSortTile);
  tile_sort_kernel<<<(unsigned)(segs * tiles), kSortThreads, 0, s>>>(keys, ids, len, tiles);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || len <= kSortTile) return e;
  double* k2 = nullptr;
  int32_t* i2 = nullptr;
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&k2), (size_t)segs * len * sizeof(double), s)) != cudaSuccess)
    return e;
  if ((e = cudaMallocAsync(reinterpret_cast<void**>(&i2), (size_t)segs * len * sizeof(int32_t), s)) != cudaSuccess)
    return e;
  double *srck = keys, *dstk = k2;
  int32_t *srci = ids, *dsti = i2;
  for (int64_t w = kSortTile; w < len; w <<= 1) {
    merge_pass_kernel<<<(unsigned)(segs * tiles), kSortThreads, 0, s>>>(srck, srci, dstk, dsti, len, w, tiles);
    count_launches(1);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    double* tk = srck;
    srck = dstk;
    dstk = tk;
    int32_t* ti = srci;
    srci = dsti;
    dsti = ti;
  }
  if (srck != keys) {
    cudaMemcpyAsync(keys, srck, (size_t)segs * len * sizeof(double), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(ids, srci, (size_t)segs * len * sizeof(int32_t), cudaMemcpyDeviceToDevice, s);
  }
  cudaFreeAsync(k2, s);
  cudaFreeAsync(i2, s);
  return cudaGetLastError();
}

}  // namespace simdex

using namespace simdex;

extern "C" int simdex_build_index(const double* items, int64_t ni, int32_t f, const double* centers,
                                  const double* theta_b, int32_t c, double* out_item_norms, int32_t* out_list_ids,
                                  double* out_bounds, int32_t* out_list_pos, void* stream) {
  SIMDEX_CHECK_ARG(items && centers && theta_b && out_item_norms && out_list_ids && out_bounds,
                   "simdex_build_index: null pointer");
  SIMDEX_CHECK_ARG(ni >= 1 && f >= 1 && c >= 1 && ni < INT32_MAX, "simdex_build_index: bad sizes");
  cudaStream_t s = as_stream(stream);
  item_norms_kernel<<<(unsigned)ceil_div(ni, 256), 256, 0, s>>>(items, ni, f, out_item_norms);
  SIMDEX_LAUNCH_CHECK("item_norms");
  Scratch<double> unit;
  SIMDEX_CUDA(unit.alloc(ni * f, s));
  unit_cols_kernel<<<(unsigned)ceil_div(ni * f, 256), 256, 0, s>>>(items, out_item_norms, ni, f, unit.p);
  SIMDEX_LAUNCH_CHECK("unit_cols");
  dim3 grid((unsigned)ceil_div(ni, 128), (unsigned)ceil_div(c, kBoundGroup));
  const size_t smem = (size_t)kBoundGroup * f * sizeof(double);
  if (smem > 48 * 1024)
    SIMDEX_CUDA(cudaFuncSetAttribute(bounds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ProfileScope _prof("bounds", s);
  bounds_kernel<<<grid, 128, smem, s>>>(unit.p, out_item_norms, ni, f, c, centers, theta_b, out_bounds,
                                        out_list_ids);
  _prof.end();
  SIMDEX_LAUNCH_CHECK("bounds");
  SIMDEX_CUDA(segmented_sort_desc(out_bounds, out_list_ids, c, ni, s));
  if (out_list_pos) {
    const int64_t tot = (int64_t)c * ni;
    list_pos_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(out_list_ids, (int64_t)c, ni, out_list_pos);
    SIMDEX_LAUNCH_CHECK("list_pos");
  }
  return SIMDEX_OK;
}

namespace simdex {
namespace {
__global__ void norm_keys_kernel(const double* __restrict__ norms, int64_t n, double* keys, int32_t* ids) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = norms[i];
  ids[i] = (int32_t)i;
}
}  // namespace
}  // namespace simdex

extern "C" int simdex_norm_order(const double* norms, int64_t n, int32_t* out_perm, void* stream) {
  SIMDEX_CHECK_ARG(norms && out_perm, "simdex_norm_order: null pointer");
  SIMDEX_CHECK_ARG(n >= 1 && n < INT32_MAX, "simdex_norm_order: bad sizes");
  cudaStream_t s = as_stream(stream);
  Scratch<double> keys;
  SIMDEX_CUDA(keys.alloc(n, s));
  norm_keys_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(norms, n, keys.p, out_perm);
  SIMDEX_LAUNCH_CHECK("norm_keys");
  SIMDEX_CUDA(segmented_sort_desc(keys.p, out_perm, 1, n, s));
  return SIMDEX_OK;
}

extern "C" int simdex_list_positions(const int32_t* list_ids, int32_t c, int64_t ni, int32_t* out_pos, void* stream) {
  SIMDEX_CHECK_ARG(list_ids && out_pos, "simdex_list_positions: null pointer");
  SIMDEX_CHECK_ARG(c >= 1 && ni >= 1, "simdex_list_positions: bad sizes");
  const int64_t tot = (int64_t)c * ni;
  list_pos_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, as_stream(stream)>>>(list_ids, (int64_t)c, ni, out_pos);
  SIMDEX_LAUNCH_CHECK("list_pos");
  return SIMDEX_OK;
}

extern "C" int simdex_max_angles(const double* users, int64_t n, int32_t f, const double* centers, int32_t c,
                                 const int64_t* assign, double* out_theta, void* stream) {
  SIMDEX_CHECK_ARG(users && centers && assign && out_theta, "simdex_max_angles: null pointer");
  SIMDEX_CHECK_ARG(n >= 1 && f >= 1 && c >= 1, "simdex_max_angles: bad sizes");
  cudaStream_t s = as_stream(stream);
  Scratch<double> cn;
  SIMDEX_CUDA(cn.alloc(c, s));
  center_norms_kernel<<<(unsigned)ceil_div(c, 128), 128, 0, s>>>(centers, c, f, cn.p);
  SIMDEX_LAUNCH_CHECK("center_norms");
  Scratch<double> unit;
  SIMDEX_CUDA(unit.alloc((size_t)c * f, s));
  unit_centers_kernel<<<(unsigned)ceil_div((int64_t)c * f, 256), 256, 0, s>>>(centers, cn.p, c, f, unit.p);
  SIMDEX_LAUNCH_CHECK("unit_centers");
  SIMDEX_CUDA(cudaMemsetAsync(out_theta, 0, sizeof(double) * c, s));
  max_angles_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(users, n, f, unit.p, cn.p, assign,
                                                               reinterpret_cast<unsigned long long*>(out_theta));
  SIMDEX_LAUNCH_CHECK("max_angles");
  return SIMDEX_OK;
}
