// SimDex index construction on device (index.py:90-155, clustering.py:65-93):
//   * per-(cluster, item) half-angle theta_ic and Eq. 2 ceiling in float64,
//   * per-cluster theta_b (max member angle) via an order-free atomic max,
//   * a batched merge sort of every cluster's list by (ceiling desc, id asc):
//     2048-element tiles bitonic-sorted in shared memory, then merge-path
//     passes over HBM/L2 (keys are unique because ids are).
#include <cfloat>
#include <cmath>

#include "common.cuh"

namespace simdex {
namespace {

constexpr int kSortThreads = 256;
constexpr int kSortTile = 2048;  // elements per shared-memory tile
constexpr int kMergeItems = 8;   // outputs per thread per merge pass

struct KV {
  double k;
  int32_t id;
};

__device__ __forceinline__ bool kv_before(double ka, int32_t ia, double kb, int32_t ib) {
  // (key desc, id asc); -0.0 == +0.0 like numpy's comparisons
  return ka > kb || (ka == kb && ia < ib);
}

__global__ void __launch_bounds__(kSortThreads) tile_sort_kernel(double* keys, int32_t* ids, int64_t len,
                                                                 int64_t tiles_per_seg) {
  __shared__ double sk[kSortTile];
  __shared__ int32_t si[kSortTile];
  const int64_t seg = blockIdx.x / tiles_per_seg, t = blockIdx.x % tiles_per_seg;
  const int64_t base = seg * len + t * kSortTile;
  const int64_t n = (len - t * kSortTile) < kSortTile ? (len - t * kSortTile) : kSortTile;
  for (int i = threadIdx.x; i < kSortTile; i += kSortThreads) {
    if (i < n) {
      sk[i] = keys[base + i];
      si[i] = ids[base + i];
    } else {
      sk[i] = -DBL_MAX;
      si[i] = INT32_MAX;
    }
  }
  for (int size = 2; size <= kSortTile; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < kSortTile / 2; i += kSortThreads) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        double ka = sk[lo], kb = sk[hi];
        int32_t ia = si[lo], ib = si[hi];
        bool swap = up ? kv_before(kb, ib, ka, ia) : kv_before(ka, ia, kb, ib);
        if (swap) {
          sk[lo] = kb;
          sk[hi] = ka;
          si[lo] = ib;
          si[hi] = ia;
        }
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kSortThreads) {
    keys[base + i] = sk[i];
    ids[base + i] = si[i];
  }
}

// Merge adjacent runs of width w inside every segment: src -> dst.
__global__ void __launch_bounds__(kSortThreads) merge_pass_kernel(const double* __restrict__ sk,
                                                                  const int32_t* __restrict__ si, double* dk,
                                                                  int32_t* di, int64_t len, int64_t w,
                                                                  int64_t chunks_per_seg, int64_t segs) {
  const int64_t gt = (int64_t)blockIdx.x * kSortThreads + threadIdx.x;
  const int64_t seg = gt / chunks_per_seg;
  if (seg >= segs) return;
  const int64_t o0 = (gt % chunks_per_seg) * kMergeItems;  // output position within segment
  if (o0 >= len) return;
  const int64_t a0 = (o0 / (2 * w)) * (2 * w);
  const int64_t la = (len - a0) < w ? (len - a0) : w;
  const int64_t b0 = a0 + la;
  const int64_t lb = (len - b0) < w ? ((len - b0) > 0 ? (len - b0) : 0) : w;
  const double* A = sk + seg * len + a0;
  const int32_t* Ai = si + seg * len + a0;
  const double* B = sk + seg * len + b0;
  const int32_t* Bi = si + seg * len + b0;
  const int64_t o = o0 - a0;  // position within the merged pair
  int64_t lo = o - lb > 0 ? o - lb : 0, hi = o < la ? o : la;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    int64_t j = o - mid - 1;
    if (kv_before(A[mid], Ai[mid], B[j], Bi[j]))
      lo = mid + 1;
    else
      hi = mid;
  }
  int64_t i = lo, j = o - lo;
  double* D = dk + seg * len + o0;
  int32_t* Di = di + seg * len + o0;
  const int64_t cnt = (len - o0) < kMergeItems ? (len - o0) : kMergeItems;
  for (int64_t t = 0; t < cnt; ++t) {
    bool takeA;
    if (i >= la)
      takeA = false;
    else if (j >= lb)
      takeA = true;
    else
      takeA = kv_before(A[i], Ai[i], B[j], Bi[j]);
    if (takeA) {
      D[t] = A[i];
      Di[t] = Ai[i];
      ++i;
    } else {
      D[t] = B[j];
      Di[t] = Bi[j];
      ++j;
    }
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

// grid: (ceil(ni/256), c).  Writes keys = ceiling, ids = item id for the sort.
__global__ void __launch_bounds__(256) bounds_kernel(const double* __restrict__ items,
                                                     const double* __restrict__ norms, int64_t ni, int f,
                                                     const double* __restrict__ centers,
                                                     const double* __restrict__ theta, double* __restrict__ keys,
                                                     int32_t* __restrict__ ids) {
  extern __shared__ double y[];  // unit centroid
  __shared__ double s_cn;
  const int c = blockIdx.y;
  const double* cen = centers + (int64_t)c * f;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < f; ++k) s = fma(cen[k], cen[k], s);
    s_cn = sqrt(s);
  }
  __syncthreads();
  const double cn = s_cn;
  for (int k = threadIdx.x; k < f; k += blockDim.x) y[k] = cn > 0.0 ? cen[k] / cn : 0.0;
  __syncthreads();
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ni) return;
  const double nrm = norms[i];
  double ang;
  if (cn == 0.0 || nrm == 0.0) {
    ang = M_PI / 2.0;
  } else {
    const double* x = items + i * f;
    double dm = 0.0, dp = 0.0;
    for (int k = 0; k < f; ++k) {
      double xk = x[k] / nrm;
      double a = xk - y[k], b = xk + y[k];
      dm = fma(a, a, dm);
      dp = fma(b, b, dp);
    }
    ang = 2.0 * atan2(sqrt(dm), sqrt(dp));
  }
  const double slack = theta[c];
  double bound = (slack < ang) ? nrm * cos(ang - slack) : nrm;
  if (bound == 0.0) bound = 0.0;  // fold -0.0
  keys[(int64_t)c * ni + i] = bound;
  ids[(int64_t)c * ni + i] = (int32_t)i;
}

// theta_b: per-user angle to its centroid, atomic max on the (non-negative) bits.
__global__ void max_angles_kernel(const double* __restrict__ users, int64_t n, int f,
                                  const double* __restrict__ centers, const double* __restrict__ cnorm,
                                  const int64_t* __restrict__ assign, unsigned long long* __restrict__ theta_bits) {
  int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t c = assign[u];
  const double* x = users + u * f;
  const double* y = centers + c * f;
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
      double xk = x[k] / un, yk = y[k] / cn;
      double a = xk - yk, b = xk + yk;
      dm = fma(a, a, dm);
      dp = fma(b, b, dp);
    }
    ang = 2.0 * atan2(sqrt(dm), sqrt(dp));
  }
  atomicMax(theta_bits + c, (unsigned long long)__double_as_longlong(ang));
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
  const int64_t chunks = ceil_div(len, kMergeItems);
  for (int64_t w = kSortTile; w < len; w <<= 1) {
    const int64_t threads = segs * chunks;
    merge_pass_kernel<<<(unsigned)ceil_div(threads, kSortThreads), kSortThreads, 0, s>>>(srck, srci, dstk, dsti,
                                                                                          len, w, chunks, segs);
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
  dim3 grid((unsigned)ceil_div(ni, 256), (unsigned)c);
  const size_t smem = (size_t)f * sizeof(double);
  if (smem > 48 * 1024) SIMDEX_CUDA(cudaFuncSetAttribute(bounds_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ProfileScope _prof("bounds", s);
  bounds_kernel<<<grid, 256, smem, s>>>(items, out_item_norms, ni, f, centers, theta_b, out_bounds, out_list_ids);
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
  SIMDEX_CUDA(cudaMemsetAsync(out_theta, 0, sizeof(double) * c, s));
  max_angles_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, s>>>(users, n, f, centers, cn.p, assign,
                                                               reinterpret_cast<unsigned long long*>(out_theta));
  SIMDEX_LAUNCH_CHECK("max_angles");
  return SIMDEX_OK;
}
