// Operand packing for the tensor-core path: float64 factors -> fp16 (scaled
// by an exact power of two, round-to-nearest-even, zero padded to [rows_pad,
// kp]) + float64 row norms; and the work-sharing prefix gather (every
// cluster's first B list items in list order, index.py:351-357).
#include <cuda_fp16.h>

#include "common.cuh"

namespace simdex {
namespace {

__global__ void pack_f16_kernel(const double* __restrict__ x, int64_t rows, int f, int scale_exp, int64_t rows_pad,
                                 int kp, uint16_t* __restrict__ out, double* __restrict__ norms) {
  // one warp per row
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows_pad) return;
  double ss = 0.0;
  for (int k = lane; k < kp; k += 32) {
    double v = (r < rows && k < f) ? x[r * f + k] : 0.0;
    ss = fma(v, v, ss);
    __half b = __double2half(ldexp(v, scale_exp));
    out[r * kp + k] = *reinterpret_cast<uint16_t*>(&b);
  }
  ss = warp_sum(ss);
  if (lane == 0 && r < rows) norms[r] = sqrt(ss);
}

// Per-row exact power-of-two scale (users): 2^e_r with max|x_r| 2^e_r in
// [1, 2), so a small-norm row keeps fp16's full relative precision instead
// of sinking into the subnormal range of a matrix-wide scale.
__global__ void pack_f16_rows_kernel(const double* __restrict__ x, int64_t rows, int f, int64_t rows_pad, int kp,
                                     uint16_t* __restrict__ out, double* __restrict__ norms,
                                     int32_t* __restrict__ row_exp) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows_pad) return;
  double m = 0.0;
  for (int k = lane; k < f; k += 32) m = fmax(m, r < rows ? fabs(x[r * f + k]) : 0.0);
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int e = m > 0.0 ? -ilogb(m) : 0;
  double ss = 0.0;
  for (int k = lane; k < kp; k += 32) {
    const double v = (r < rows && k < f) ? x[r * f + k] : 0.0;
    ss = fma(v, v, ss);
    __half b = __double2half(ldexp(v, e));
    out[r * kp + k] = *reinterpret_cast<uint16_t*>(&b);
  }
  ss = warp_sum(ss);
  if (lane == 0 && r < rows) {
    norms[r] = sqrt(ss);
    row_exp[r] = e;
  }
}

__global__ void gather_prefix_kernel(const uint16_t* __restrict__ ib, const double* __restrict__ inorm, int64_t ni,
                                     int kp, const int32_t* __restrict__ list_ids, int64_t bp, int64_t b_pad,
                                     int64_t n_clusters, uint16_t* __restrict__ out, double* __restrict__ onorm) {
  // one thread per 16-byte piece of a (cluster, prefix row): the stores of a
  // warp are contiguous (a warp per row kept 8 of 32 lanes busy at kp = 64)
  const int vpr = kp / 8;
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t row = g / vpr;
  const int v = (int)(g - row * vpr);
  const int64_t c = row / b_pad, r = row - c * b_pad;
  if (c >= n_clusters) return;
  const bool live = r < bp;
  const int64_t src = live ? list_ids[c * ni + r] : 0;
  reinterpret_cast<uint4*>(out)[g] = live ? reinterpret_cast<const uint4*>(ib + src * kp)[v] : make_uint4(0, 0, 0, 0);
  if (v == 0) onorm[row] = live ? inorm[src] : 0.0;
}

// Ordering keys of a cluster's prefix: the centroid's float64 score c . i of
// each of its first bp list items.  One lane per (cluster, position), the
// cluster's centre in shared memory, the item row read by its lane (the
// catalogue sits in L2); grid = (chunks of 256 positions, clusters).  (A warp
// per position spent 60 instructions per key on the strided partials and the
// shuffle tree: 0.265 ms for 256 x 4,096 keys at cfg2.)
__global__ void __launch_bounds__(256) prefix_keys_kernel(const int32_t* __restrict__ list_ids, int64_t ni,
                                                          int64_t bp, const double* __restrict__ centers,
                                                          const double* __restrict__ items, int f,
                                                          int64_t n_clusters, double* __restrict__ keys,
                                                          int32_t* __restrict__ ids) {
  extern __shared__ double cen[];  // [f]
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t c = blockIdx.y; c < n_clusters; c += gridDim.y) {
  __syncthreads();
  for (int q = threadIdx.x; q < f; q += blockDim.x) cen[q] = centers[c * f + q];
  __syncthreads();
  if (j >= bp) continue;
  const int32_t id = list_ids[c * ni + j];
  const double* x = items + (int64_t)id * f;
  double a0 = 0.0, a1 = 0.0;
  int q = 0;
  if ((f & 1) == 0) {  // rows of an even f are 16-byte aligned
    const double2* x2 = reinterpret_cast<const double2*>(x);
#pragma unroll 5
    for (; q + 1 < f; q += 2) {
      const double2 v = x2[q >> 1];
      a0 = fma(cen[q], v.x, a0);
      a1 = fma(cen[q + 1], v.y, a1);
    }
  }
  for (; q < f; ++q) a0 = fma(cen[q], x[q], a0);
  keys[c * bp + j] = a0 + a1;
  ids[c * bp + j] = id;
  }
}

// Per 128-item tile of the reordered prefix: the largest list ceiling at or
// after the tile (the early-exit bound, index.py:90-100), unscaled.  One CTA
// per cluster: a warp per tile takes the tile's maximum, then a suffix scan.
__global__ void __launch_bounds__(1024) prefix_tile_ceil_kernel(const int32_t* __restrict__ ids, int64_t bp,
                                                                int64_t b_pad, const int32_t* __restrict__ list_pos,
                                                                const double* __restrict__ bounds, int64_t ni,
                                                                double* __restrict__ tile_ceil) {
  extern __shared__ double tmax[];  // [tiles]
  const int64_t c = blockIdx.x;
  const int tiles = (int)(b_pad / 128);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int t = w; t < tiles; t += nw) {
    double m = 0.0;
    for (int64_t j = (int64_t)t * 128 + lane; j < (int64_t)(t + 1) * 128 && j < bp; j += 32) {
      const int32_t id = ids[c * bp + j];
      m = fmax(m, bounds[c * ni + list_pos[c * ni + id]]);
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) tmax[t] = m;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double m = 0.0;
    for (int t = tiles - 1; t >= 0; --t) {
      m = fmax(m, tmax[t]);
      tile_ceil[c * tiles + t] = m;
    }
  }
}

__global__ void max_abs_kernel(const double* __restrict__ x, int64_t n, unsigned long long* __restrict__ out) {
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(x[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));  // m >= 0
}

}  // namespace

int launch_max_abs(const double* x, int64_t n, double* out, cudaStream_t s) {
  SIMDEX_CUDA(cudaMemsetAsync(out, 0, sizeof(double), s));
  if (n == 0) return SIMDEX_OK;
  int64_t blocks = ceil_div(n, 256);
  if (blocks > 4 * 148) blocks = 4 * 148;
  max_abs_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, n, reinterpret_cast<unsigned long long*>(out));
  SIMDEX_LAUNCH_CHECK("max_abs");
  return SIMDEX_OK;
}

int launch_pack_f16(const double* x, int64_t rows, int32_t f, int32_t scale_exp, int64_t rows_pad, int32_t kp,
                     uint16_t* out, double* norms, cudaStream_t s) {
  pack_f16_kernel<<<(unsigned)ceil_div(rows_pad, 8), 256, 0, s>>>(x, rows, f, scale_exp, rows_pad, kp, out, norms);
  SIMDEX_LAUNCH_CHECK("pack_f16");
  return SIMDEX_OK;
}

int launch_pack_f16_rows(const double* x, int64_t rows, int32_t f, int64_t rows_pad, int32_t kp, uint16_t* out,
                         double* norms, int32_t* row_exp, cudaStream_t s) {
  pack_f16_rows_kernel<<<(unsigned)ceil_div(rows_pad, 8), 256, 0, s>>>(x, rows, f, rows_pad, kp, out, norms, row_exp);
  SIMDEX_LAUNCH_CHECK("pack_f16_rows");
  return SIMDEX_OK;
}

int launch_gather_prefix(const uint16_t* ib, const double* i_norm, int64_t ni, int32_t kp, const int32_t* list_ids,
                         int32_t c, int64_t block, int64_t b_pad, uint16_t* out, double* onorm, cudaStream_t s) {
  const int64_t bp = block < ni ? block : ni;
  const int64_t pieces = (int64_t)c * b_pad * (kp / 8);
  gather_prefix_kernel<<<(unsigned)ceil_div(pieces, 256), 256, 0, s>>>(ib, i_norm, ni, kp, list_ids, bp, b_pad, c,
                                                                       out, onorm);
  SIMDEX_LAUNCH_CHECK("gather_prefix");
  return SIMDEX_OK;
}

// Work-sharing prefix in "likely score" order: each cluster's first B' list
// items sorted by the centroid's score (desc, id asc), so a cluster's users
// meet their best items in the first chunks and their thresholds rise at
// once (the stage-1 appends concentrate early in list order).  The prefix
// top-K and visited do not depend on the order in which the prefix is scored.
// Hybrid order: a cluster's `head` best prefix items by the centroid's score
// first (the thresholds rise at once), then the rest of the prefix in list
// (ceiling) order, so the per-tile suffix maxima of the ceilings fall like
// the list's and the early exit can stop a warp inside the tail.  One CTA per
// cluster: head items marked by list position, the tail compacted in list
// order by a CTA scan.
__global__ void __launch_bounds__(1024) prefix_hybrid_kernel(const int32_t* __restrict__ sorted, int64_t bp,
                                                             int64_t head, const int32_t* __restrict__ list_ids,
                                                             const int32_t* __restrict__ list_pos, int64_t ni,
                                                             int32_t* __restrict__ out) {
  extern __shared__ unsigned char flag[];  // [bp]
  __shared__ int wsum[32];
  const int64_t c = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  for (int64_t p = t; p < bp; p += blockDim.x) flag[p] = 0;
  __syncthreads();
  for (int64_t i = t; i < head; i += blockDim.x) {
    const int32_t id = sorted[c * bp + i];
    flag[list_pos[c * ni + id]] = 1;
    out[c * bp + i] = id;
  }
  __syncthreads();
  // tail: list positions without a flag, in order (chunks of blockDim.x positions)
  int64_t base = head;
  for (int64_t p0 = 0; p0 < bp; p0 += blockDim.x) {
    const int64_t p = p0 + t;
    const int keep = (p < bp && !flag[p]) ? 1 : 0;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wsum[w] = __popc(bal);
    __syncthreads();
    int before = 0, tot = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
      if (q < w) before += wsum[q];
      tot += wsum[q];
    }
    if (keep) out[c * bp + base + before + __popc(bal & ((1u << lane) - 1u))] = list_ids[c * ni + p];
    base += tot;
    __syncthreads();
  }
}

int launch_build_prefix_ordered(const uint16_t* ib, const double* i_norm, int64_t ni, int32_t kp,
                                const double* items, int32_t f, const double* centers,
                                const int32_t* list_ids, const int32_t* list_pos, const double* bounds, int32_t c,
                                int64_t block, int64_t b_pad, uint16_t* out, double* onorm, int32_t* out_ids,
                                double* out_tile_ceil, cudaStream_t s, int64_t head) {
  const int64_t bp = block < ni ? block : ni;
  Scratch<double> keys;
  SIMDEX_CUDA(keys.alloc((size_t)c * bp, s));
  int32_t* ids = out_ids;  // [c, bp] sorted in place, then spread to [c, b_pad]
  Scratch<int32_t> tmp;
  SIMDEX_CUDA(tmp.alloc((size_t)c * bp, s));
  prefix_keys_kernel<<<dim3((unsigned)ceil_div(bp, 256), (unsigned)(c < 65535 ? c : 65535)), 256,
                       sizeof(double) * f, s>>>(list_ids, ni, bp, centers, items, f, c, keys.p, tmp.p);
  SIMDEX_LAUNCH_CHECK("prefix_keys");
  SIMDEX_CUDA(segmented_sort_desc(keys.p, tmp.p, c, bp, s));
  Scratch<int32_t> hyb;
  if (head > 0 && head < bp && bp <= 48 * 1024) {
    SIMDEX_CUDA(hyb.alloc((size_t)c * bp, s));
    prefix_hybrid_kernel<<<(unsigned)c, 1024, (size_t)bp, s>>>(tmp.p, bp, head, list_ids, list_pos, ni, hyb.p);
    SIMDEX_LAUNCH_CHECK("prefix_hybrid");
    SIMDEX_CUDA(cudaMemcpyAsync(tmp.p, hyb.p, sizeof(int32_t) * (size_t)c * bp, cudaMemcpyDeviceToDevice, s));
  }
  const size_t tsm = (size_t)(b_pad / 128) * sizeof(double);
  if (tsm > 48 * 1024) {
    set_error("simdex_build_prefix_ordered: prefix longer than %d tiles", 48 * 1024 / 8);
    return SIMDEX_EUNSUPPORTED;
  }
  prefix_tile_ceil_kernel<<<(unsigned)c, 1024, tsm, s>>>(tmp.p, bp, b_pad, list_pos, bounds, ni, out_tile_ceil);
  SIMDEX_LAUNCH_CHECK("prefix_tile_ceil");
  // gather the operand rows in the new order (the sorted ids act as a list of length bp)
  const int64_t pieces = (int64_t)c * b_pad * (kp / 8);
  gather_prefix_kernel<<<(unsigned)ceil_div(pieces, 256), 256, 0, s>>>(ib, i_norm, bp, kp, tmp.p, bp, b_pad, c, out,
                                                                       onorm);
  SIMDEX_LAUNCH_CHECK("gather_prefix");
  SIMDEX_CUDA(cudaMemsetAsync(ids, 0xff, sizeof(int32_t) * (size_t)c * b_pad, s));
  SIMDEX_CUDA(cudaMemcpy2DAsync(ids, sizeof(int32_t) * b_pad, tmp.p, sizeof(int32_t) * bp, sizeof(int32_t) * bp, c,
                                cudaMemcpyDeviceToDevice, s));
  return SIMDEX_OK;
}

}  // namespace simdex
