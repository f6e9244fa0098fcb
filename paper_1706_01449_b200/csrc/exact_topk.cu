// Exact float64 top-K: the GPU form of the reference oracle topk_naive
// (brute.py:43-56) and the certified fallback of the tensor-core path.
//
//   1. fp64 SIMT tile GEMM writes a [rows_batch, ni] score block to HBM;
//   2. one CTA per row radix-selects the k-th best 64-bit ordered key
//      (8 passes of 8 bits over the row, L2 resident), gathers the strictly
//      better entries plus the lowest-id ties, and bitonic-sorts them in
//      shared memory by (score desc, id asc)  (index.py:158-163);
//   3. k > kSelectMax sorts whole rows with the segmented merge sort.
#include <cfloat>

#include "common.cuh"

namespace simdex {
namespace {

constexpr int kTile = 64;      // rows x items per CTA
constexpr int kKc = 16;        // factor chunk
constexpr int kSelectMax = 4096;

// S[r, j] = users[rows[r]] . items[j]   (rows == nullptr: row r0 + r)
__global__ void __launch_bounds__(256) score_f64_kernel(const double* __restrict__ users,
                                                        const int64_t* __restrict__ rows, int64_t r0,
                                                        int64_t nr, const double* __restrict__ items,
                                                        int64_t ni, int f, double* __restrict__ S) {
  __shared__ double As[kKc][kTile + 1];
  __shared__ double Bs[kKc][kTile + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t rbase = (int64_t)blockIdx.y * kTile, cbase = (int64_t)blockIdx.x * kTile;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < f; k0 += kKc) {
    for (int e = threadIdx.x; e < kTile * kKc; e += 256) {
      int rr = e / kKc, kk = e % kKc;
      int64_t r = rbase + rr;
      double a = 0.0;
      if (r < nr && k0 + kk < f) {
        int64_t ur = rows ? rows[r0 + r] : (r0 + r);
        a = users[ur * f + k0 + kk];
      }
      As[kk][rr] = a;
      int64_t c = cbase + rr;
      Bs[kk][rr] = (c < ni && k0 + kk < f) ? items[c * f + k0 + kk] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kKc; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t r = rbase + ty + 16 * i;
    if (r >= nr) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t c = cbase + tx + 16 * j;
      if (c < ni) S[r * ni + c] = acc[i][j];
    }
  }
}

struct Entry {
  double s;
  int32_t id;
};

__device__ __forceinline__ bool entry_before(const Entry& a, const Entry& b) {
  return ranks_before(a.s, a.id, b.s, b.id);
}

// In-place bitonic sort of n (power of two) entries in shared memory,
// "before" entries first.
__device__ void block_bitonic(Entry* e, int n) {
  for (int size = 2; size <= n; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < n / 2; i += blockDim.x) {
        int lo = 2 * i - (i & (stride - 1));
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        Entry a = e[lo], b = e[hi];
        bool swap = up ? entry_before(b, a) : entry_before(a, b);
        if (swap) {
          e[lo] = b;
          e[hi] = a;
        }
      }
    }
  }
  __syncthreads();
}

// The calling CTA's exact top-k_eff of row[0, ni) into out_ids / out_scores
// [k_eff] (buf: pow2 entries of shared memory).
__device__ void select_row_block(const double* __restrict__ row, int64_t ni, int k_eff, int pow2, Entry* buf,
                                 int32_t* __restrict__ o_ids, double* __restrict__ o_scores) {
  __shared__ uint32_t hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int s_need;
  __shared__ int s_nlt, s_neq_base;
  __shared__ int warp_cnt[8];

  uint64_t prefix = 0, mask = 0;
  int need = k_eff;  // rank (1-based) of the wanted key among keys matching prefix
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (int64_t j = threadIdx.x; j < ni; j += blockDim.x) {
      uint64_t key = desc_key(row[j]);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t cum = 0;
      int d = 0;
      for (; d < 256; ++d) {
        if (cum + hist[d] >= (uint32_t)need) break;
        cum += hist[d];
      }
      s_need = need - (int)cum;
      s_prefix = prefix | ((uint64_t)d << shift);
    }
    __syncthreads();
    need = s_need;
    prefix = s_prefix;
    mask |= (0xffull << shift);
    __syncthreads();
  }
  // prefix = key of the k-th best; `need` ties with that key are taken (lowest ids).
  if (threadIdx.x == 0) {
    s_nlt = 0;
    s_neq_base = 0;
  }
  __syncthreads();
  for (int64_t j = threadIdx.x; j < ni; j += blockDim.x) {
    double v = row[j];
    if (desc_key(v) < prefix) {
      int p = atomicAdd(&s_nlt, 1);
      buf[p] = Entry{v, (int32_t)j};
    }
  }
  __syncthreads();
  const int nlt = s_nlt;  // == k_eff - need
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t j0 = 0; j0 < ni; j0 += blockDim.x) {
    int64_t j = j0 + threadIdx.x;
    bool eq = (j < ni) && desc_key(row[j]) == prefix;
    unsigned bal = __ballot_sync(0xffffffffu, eq);
    if (lane == 0) warp_cnt[wid] = __popc(bal);
    __syncthreads();
    int before = s_neq_base;
    for (int w = 0; w < wid; ++w) before += warp_cnt[w];
    before += __popc(bal & ((1u << lane) - 1u));
    if (eq && before < need) buf[nlt + before] = Entry{row[j], (int32_t)j};
    __syncthreads();
    if (threadIdx.x == 0) {
      int tot = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += warp_cnt[w];
      s_neq_base += tot;
    }
    __syncthreads();
    if (s_neq_base >= need) break;
  }
  for (int i = k_eff + threadIdx.x; i < pow2; i += blockDim.x) buf[i] = Entry{-DBL_MAX, INT32_MAX};
  block_bitonic(buf, pow2);
  for (int i = threadIdx.x; i < k_eff; i += blockDim.x) {
    o_ids[i] = buf[i].id;
    o_scores[i] = buf[i].s;
  }
  __syncthreads();
}

// One CTA per row: exact top-k_eff of S[row, :ni].
__global__ void __launch_bounds__(256) select_rows_kernel(const double* __restrict__ S, int64_t ni, int k_eff,
                                                          int pow2, int32_t* __restrict__ out_ids,
                                                          double* __restrict__ out_scores, int64_t out_row0,
                                                          const int64_t* __restrict__ out_map) {
  extern __shared__ unsigned char smem_raw[];
  Entry* buf = reinterpret_cast<Entry*>(smem_raw);
  const int64_t orow = out_map ? out_map[out_row0 + blockIdx.x] : out_row0 + blockIdx.x;
  const int64_t o = orow * (int64_t)k_eff;
  select_row_block(S + (int64_t)blockIdx.x * ni, ni, k_eff, pow2, buf, out_ids + o, out_scores + o);
}

// Device-counted rows (the tensor-core passes' band-overflow fallback): a
// persistent CTA per slab row scores its user against every item in float64
// (factor order, like score_f64_kernel) into the slab, then selects.
template <class U, class I>
__global__ void __launch_bounds__(256) exact_rows_dev_kernel(const U* __restrict__ users, const I* __restrict__ items,
                                                             int64_t ni, int f, const int64_t* __restrict__ rows,
                                                             const int64_t* __restrict__ user_of,
                                                             const int32_t* __restrict__ n_rows, int k_eff, int pow2,
                                                             const int64_t* __restrict__ out_map,
                                                             int32_t* __restrict__ out_ids,
                                                             double* __restrict__ out_scores, double* __restrict__ slab) {
  extern __shared__ unsigned char smem_raw[];
  Entry* buf = reinterpret_cast<Entry*>(smem_raw);
  double* urow = reinterpret_cast<double*>(smem_raw + (size_t)pow2 * sizeof(Entry));
  const int n = *n_rows;
  double* row = slab + (int64_t)blockIdx.x * ni;
  for (int r = blockIdx.x; r < n; r += gridDim.x) {
    int64_t u = rows[r];
    if (user_of) u = user_of[u];
    for (int q = threadIdx.x; q < f; q += blockDim.x) urow[q] = (double)users[u * f + q];
    __syncthreads();
    for (int64_t j = threadIdx.x; j < ni; j += blockDim.x) {
      const I* x = items + j * f;
      double acc = 0.0;
      for (int q = 0; q < f; ++q) acc = fma(urow[q], (double)x[q], acc);
      row[j] = acc;
    }
    __syncthreads();
    const int64_t o = out_map[r] * (int64_t)k_eff;
    select_row_block(row, ni, k_eff, pow2, buf, out_ids + o, out_scores + o);
  }
}

__global__ void iota_rows_kernel(int32_t* ids, int64_t rows, int64_t n) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < rows * n) ids[t] = (int32_t)(t % n);
}

__global__ void take_prefix_kernel(const double* S, const int32_t* ids, int64_t rows, int64_t n, int k,
                                   int32_t* out_ids, double* out_scores, int64_t out_row0, const int64_t* out_map) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * k) return;
  int64_t r = t / k, i = t % k;
  const int64_t o = out_map ? out_map[out_row0 + r] : out_row0 + r;
  out_ids[o * k + i] = ids[r * n + i];
  out_scores[o * k + i] = S[r * n + i];
}

// ---------------------------------------------------------------------------
// merge of per-shard sorted lists: one warp per user
// ---------------------------------------------------------------------------
__global__ void merge_lists_kernel(const int32_t* __restrict__ in_ids, const double* __restrict__ in_sc,
                                   int parts, int64_t nu, int kk, int k_out, int32_t* __restrict__ out_ids,
                                   double* __restrict__ out_sc) {
  int64_t u = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (u >= nu) return;
  int pos = 0;  // lane p < parts: head position of list p
  for (int o = 0; o < k_out; ++o) {
    double s = -DBL_MAX;
    int32_t id = INT32_MAX;
    bool live = lane < parts && pos < kk;
    if (live) {
      int64_t at = ((int64_t)lane * nu + u) * kk + pos;
      s = in_sc[at];
      id = in_ids[at];
      if (id < 0) live = false, s = -DBL_MAX, id = INT32_MAX;  // padded slot
    }
    int src = lane;
    for (int off = 16; off > 0; off >>= 1) {
      double s2 = __shfl_xor_sync(0xffffffffu, s, off);
      int32_t i2 = __shfl_xor_sync(0xffffffffu, id, off);
      int src2 = __shfl_xor_sync(0xffffffffu, src, off);
      if (ranks_before(s2, i2, s, id) || (s2 == s && i2 == id && src2 < src)) {
        s = s2;
        id = i2;
        src = src2;
      }
    }
    if (lane == 0) {
      out_ids[u * k_out + o] = id == INT32_MAX ? -1 : id;
      out_sc[u * k_out + o] = s;
    }
    if (lane == src) ++pos;
  }
}

}  // namespace

int exact_topk_rows(const double* users, const double* items, int64_t ni, int32_t f, const int64_t* rows,
                    int64_t n_rows, int32_t k, int32_t* out_ids, double* out_scores, cudaStream_t s) {
  return exact_topk_rows_mapped(users, items, ni, f, rows, n_rows, k, nullptr, out_ids, out_scores, s);
}

int exact_topk_rows_mapped(const double* users, const double* items, int64_t ni, int32_t f, const int64_t* rows,
                           int64_t n_rows, int32_t k, const int64_t* out_map, int32_t* out_ids, double* out_scores,
                           cudaStream_t s) {
  const int k_eff = (int)(k < ni ? k : ni);
  if (n_rows == 0) return SIMDEX_OK;
  // score block budget ~1 GiB
  int64_t rb = (int64_t(1) << 27) / (ni > 0 ? ni : 1);
  if (rb < 1) rb = 1;
  if (rb > n_rows) rb = n_rows;
  Scratch<double> S;
  SIMDEX_CUDA(S.alloc((size_t)rb * ni, s));
  Scratch<int32_t> ids;
  const bool full_sort = k_eff > kSelectMax;
  if (full_sort) SIMDEX_CUDA(ids.alloc((size_t)rb * ni, s));
  int pow2 = 1;
  while (pow2 < k_eff) pow2 <<= 1;
  const size_t smem = (size_t)pow2 * sizeof(Entry);
  if (!full_sort && smem > 48 * 1024)
    SIMDEX_CUDA(cudaFuncSetAttribute(select_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  for (int64_t r0 = 0; r0 < n_rows; r0 += rb) {
    int64_t nr = (n_rows - r0 < rb) ? n_rows - r0 : rb;
    dim3 grid((unsigned)ceil_div(ni, kTile), (unsigned)ceil_div(nr, kTile));
    ProfileScope _prof("score_f64", s);
    score_f64_kernel<<<grid, 256, 0, s>>>(users, rows, r0, nr, items, ni, f, S.p);
    _prof.end();
    SIMDEX_LAUNCH_CHECK("score_f64");
    if (!full_sort) {
      ProfileScope _prof("select_rows", s);
      select_rows_kernel<<<(unsigned)nr, 256, smem, s>>>(S.p, ni, k_eff, pow2, out_ids, out_scores, r0,
                                                                          out_map);
      _prof.end();
      SIMDEX_LAUNCH_CHECK("select_rows");
    } else {
      int64_t tot = nr * ni;
      iota_rows_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(ids.p, nr, ni);
      SIMDEX_LAUNCH_CHECK("iota");
      SIMDEX_CUDA(segmented_sort_desc(S.p, ids.p, nr, ni, s));
      take_prefix_kernel<<<(unsigned)ceil_div(nr * k_eff, 256), 256, 0, s>>>(S.p, ids.p, nr, ni, k_eff, out_ids,
                                                                            out_scores, r0, out_map);
      SIMDEX_LAUNCH_CHECK("take_prefix");
    }
  }
  return SIMDEX_OK;
}

int exact_slab_ctas(int64_t ni) {
  int64_t g = (int64_t(32) << 20) / (ni > 0 ? ni : 1);  // 256 MB of float64 rows
  const int64_t mx = 2 * (int64_t)sm_count();
  return (int)(g < 1 ? 1 : g > mx ? mx : g);
}

int exact_topk_devcount(const double* users, const float* users32, const double* items, const float* items32,
                        int64_t ni, int32_t f, const int64_t* rows, const int64_t* user_of, const int32_t* n_rows,
                        int32_t k, const int64_t* out_map, int32_t* out_ids, double* out_scores, double* slab,
                        cudaStream_t s) {
  const int k_eff = (int)(k < ni ? k : ni);
  int pow2 = 1;
  while (pow2 < k_eff) pow2 <<= 1;
  const size_t smem = (size_t)pow2 * sizeof(Entry) + (size_t)f * sizeof(double);
  if (smem > 200 * 1024) {
    set_error("exact fallback: k_eff %d / f %d too large", k_eff, f);
    return SIMDEX_EUNSUPPORTED;
  }
  const int grid = exact_slab_ctas(ni);
#define SIMDEX_EXACT_DEV(U, I, uu, ii)                                                                       \
  do {                                                                                                     \
    if (smem > 48 * 1024)                                                                                  \
      SIMDEX_CUDA(cudaFuncSetAttribute(exact_rows_dev_kernel<U, I>,                                        \
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));           \
    exact_rows_dev_kernel<U, I><<<grid, 256, smem, s>>>(uu, ii, ni, f, rows, user_of, n_rows, k_eff, pow2,  \
                                                        out_map, out_ids, out_scores, slab);               \
  } while (0)
  if (users32 && items32)
    SIMDEX_EXACT_DEV(float, float, users32, items32);
  else if (users32)
    SIMDEX_EXACT_DEV(float, double, users32, items);
  else if (items32)
    SIMDEX_EXACT_DEV(double, float, users, items32);
  else
    SIMDEX_EXACT_DEV(double, double, users, items);
#undef SIMDEX_EXACT_DEV
  SIMDEX_LAUNCH_CHECK("exact_rows_dev");
  return SIMDEX_OK;
}

int merge_lists(const int32_t* in_ids, const double* in_scores, int32_t parts, int64_t nu, int32_t kk,
                int32_t k_out, int32_t* out_ids, double* out_scores, cudaStream_t s) {
  if (nu == 0) return SIMDEX_OK;
  merge_lists_kernel<<<(unsigned)ceil_div(nu, 8), 256, 0, s>>>(in_ids, in_scores, parts, nu, kk, k_out, out_ids,
                                                               out_scores);
  SIMDEX_LAUNCH_CHECK("merge_lists");
  return SIMDEX_OK;
}

}  // namespace simdex
