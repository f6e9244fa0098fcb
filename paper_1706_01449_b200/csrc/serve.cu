// Serving entry points: topk_matmul (brute.py:59-113), work-sharing
// query_batch (index.py:305-389) and the query grouping it needs.
#include "common.cuh"

namespace simdex {
int gemm_topk_brute(const double* users, const float* users32, const uint16_t* ub, const double* u_norm, int64_t nu, const double* items,
                    const float* items32, const uint16_t* ib, const double* i_norm, const int32_t* item_perm, int64_t ib_rows, int64_t ni,
                    int32_t f, int32_t kp, int32_t su, const int32_t* u_exp, int32_t si, int32_t k, int32_t* out_ids,
                    double* out_scores, int64_t* heap_ops, float* debug_out, int32_t options, Ctx* ctx,
                    cudaStream_t s);
int gemm_topk_ws(const double* users, const float* users32, const uint16_t* ub, const double* unorm, int64_t nu, const double* items,
                 const float* items32, const uint16_t* ib, const double* i_norm, const int32_t* item_perm, int64_t ib_rows, int64_t ni,
                 int32_t f, int32_t kp, int32_t su, const int32_t* u_exp, int32_t si,
                 const int32_t* list_ids, const int32_t* list_pos, const double* bounds, int32_t c, int64_t block,
                 const uint16_t* prefix_b, const double* prefix_norm, const int32_t* prefix_ids,
                 const double* prefix_tile_ceil, int64_t b_pad, const int64_t* q_user,
                 const int64_t* q_perm, const int64_t* q_off, int64_t nq, int32_t k, int32_t* out_ids,
                 double* out_scores, int64_t* out_visited, int32_t options, Ctx* ctx, cudaStream_t s);

void read_ws_stats(int64_t* out);
int64_t read_fallback_count();
void read_pairs(int64_t* out2);

namespace {
constexpr int kMaxMatmulK = 256;
constexpr int kMaxKp = 256;

// label of each query position: its user's cluster
__global__ void query_labels_kernel(const int64_t* __restrict__ q_user, int64_t nq, const int64_t* __restrict__ assign,
                                    int64_t* __restrict__ labels) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nq) labels[i] = assign[q_user[i]];
}

__global__ void gather_users_kernel(const int64_t* __restrict__ perm, const int64_t* __restrict__ q_user, int64_t nq,
                                    int64_t* __restrict__ out_q) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < nq) out_q[j] = q_user[perm[j]];
}
}  // namespace
}  // namespace simdex

using namespace simdex;

extern "C" int simdex_topk_matmul_ctx(void* ctx, const double* users, const float* users32, const uint16_t* ub,
                                      const double* u_norm, int64_t nu, const double* items, const float* items32,
                                      const uint16_t* ib, const double* i_norm, const int32_t* item_perm,
                                      int64_t ib_rows, int64_t ni, int32_t f, int32_t kp, int32_t su,
                                      const int32_t* u_row_exp, int32_t si, int32_t k, int32_t* out_ids,
                                      double* out_scores, int64_t* heap_ops, int32_t options, void* stream) {
  SIMDEX_CHECK_ARG(users && items && out_ids && out_scores, "simdex_topk_matmul: null pointer");
  SIMDEX_CHECK_ARG(nu >= 1 && ni >= 1 && f >= 1 && k >= 1 && ni < INT32_MAX, "simdex_topk_matmul: bad sizes");
  const int64_t k_eff = k < ni ? k : ni;
  if (k_eff > kMaxMatmulK || kp > kMaxKp || !ub || !ib || !u_norm || !i_norm) {
    // outside the tensor-core path's envelope: the exact float64 scan gives the same answer
    if (heap_ops) SIMDEX_CUDA(cudaMemsetAsync(heap_ops, 0, sizeof(int64_t) * nu, as_stream(stream)));
    return exact_topk_rows(users, items, ni, f, nullptr, nu, k, out_ids, out_scores, as_stream(stream));
  }
  SIMDEX_CHECK_ARG(kp % 64 == 0 && kp >= f, "simdex_topk_matmul: kp must be a multiple of 64 >= f");
  Ctx* c = ctx_or_default(ctx);
  SIMDEX_CHECK_ARG(c, "simdex_topk_matmul: no execution context");
  return gemm_topk_brute(users, users32, ub, u_norm, nu, items, items32, ib, i_norm, item_perm, ib_rows, ni, f, kp, su,
                         u_row_exp, si, k, out_ids, out_scores, heap_ops, nullptr, options, c, as_stream(stream));
}

extern "C" int simdex_topk_matmul(const double* users, const float* users32, const uint16_t* ub, const double* u_norm, int64_t nu,
                                  const double* items, const float* items32, const uint16_t* ib, const double* i_norm,
                                  const int32_t* item_perm, int64_t ib_rows, int64_t ni, int32_t f, int32_t kp,
                                  int32_t su, int32_t si, int32_t k, int32_t* out_ids, double* out_scores,
                                  int64_t* heap_ops, void* stream) {
  return simdex_topk_matmul_ctx(nullptr, users, users32, ub, u_norm, nu, items, items32, ib, i_norm, item_perm, ib_rows,
                                ni, f, kp, su, nullptr, si, k, out_ids, out_scores, heap_ops, SIMDEX_MM_NORM_AUTO,
                                stream);
}

extern "C" int simdex_fallback_rows(int64_t* out) {
  SIMDEX_CHECK_ARG(out, "simdex_fallback_rows: null pointer");
  *out = read_fallback_count();
  return SIMDEX_OK;
}

extern "C" int simdex_executed_pairs(int64_t* out2) {
  SIMDEX_CHECK_ARG(out2, "simdex_executed_pairs: null pointer");
  read_pairs(out2);
  return SIMDEX_OK;
}

extern "C" int simdex_ctx_stats(void* ctx, int64_t* out4) {
  SIMDEX_CHECK_ARG(out4, "simdex_ctx_stats: null pointer");
  Ctx* c = ctx_or_default(ctx);
  if (!c) return SIMDEX_ECUDA;
  const int64_t* h = ctx_host_slots(c);
  out4[0] = (int64_t)(int32_t)(h[0] & 0xffffffffll);
  out4[1] = h[1];
  out4[2] = h[2];
  out4[3] = h[3];
  return SIMDEX_OK;
}

extern "C" int simdex_ws_stats(int64_t* out5) {
  SIMDEX_CHECK_ARG(out5, "simdex_ws_stats: null pointer");
  read_ws_stats(out5);
  return SIMDEX_OK;
}

extern "C" int simdex_gemm_debug(const uint16_t* ub, int64_t nu, const uint16_t* ib, int64_t ni, int32_t f,
                                 int32_t kp, float* out, void* stream) {
  SIMDEX_CHECK_ARG(ub && ib && out, "simdex_gemm_debug: null pointer");
  SIMDEX_CHECK_ARG(nu >= 1 && ni >= 1 && f >= 1 && kp % 64 == 0 && kp >= f && kp <= kMaxKp,
                   "simdex_gemm_debug: bad sizes");
  cudaStream_t s = as_stream(stream);
  Scratch<double> un, in;
  SIMDEX_CUDA(un.alloc(nu, s));
  SIMDEX_CUDA(in.alloc(ni, s));
  SIMDEX_CUDA(cudaMemsetAsync(un.p, 0, sizeof(double) * nu, s));
  SIMDEX_CUDA(cudaMemsetAsync(in.p, 0, sizeof(double) * ni, s));
  return gemm_topk_brute(nullptr, nullptr, ub, un.p, nu, nullptr, nullptr, ib, in.p, nullptr, 0, ni, f, kp, 0, nullptr, 0, 1,
                         nullptr, nullptr, nullptr, out, 0, ctx_or_default(nullptr), s);
}

extern "C" int simdex_group_queries(const int64_t* q_user, int64_t nq, const int64_t* assign, int32_t c,
                                    int64_t* out_q_user, int64_t* out_perm, int64_t* out_off, void* stream) {
  SIMDEX_CHECK_ARG(q_user && assign && out_q_user && out_perm && out_off, "simdex_group_queries: null pointer");
  SIMDEX_CHECK_ARG(nq >= 0 && nq < INT32_MAX && c >= 1, "simdex_group_queries: bad sizes");
  cudaStream_t s = as_stream(stream);
  // (cluster, query position) order by a stable counting sort
  Scratch<int64_t> labels, counts;
  SIMDEX_CUDA(labels.alloc(nq > 0 ? nq : 1, s));
  SIMDEX_CUDA(counts.alloc(c, s));
  if (nq > 0) {
    query_labels_kernel<<<(unsigned)ceil_div(nq, 256), 256, 0, s>>>(q_user, nq, assign, labels.p);
    SIMDEX_LAUNCH_CHECK("query_labels");
  }
  SIMDEX_CUDA(group_stable(labels.p, nq, c, counts.p, out_perm, out_off, s));
  if (nq > 0) {
    gather_users_kernel<<<(unsigned)ceil_div(nq, 256), 256, 0, s>>>(out_perm, q_user, nq, out_q_user);
    SIMDEX_LAUNCH_CHECK("gather_users");
  }
  return SIMDEX_OK;
}

extern "C" int simdex_query_ws_ctx(void* ctx, const double* users, const float* users32, const uint16_t* ub, const double* user_norms, int64_t nu,
                               const double* items, const float* items32, const uint16_t* ib,
                               const double* item_norms,
                               const int32_t* item_perm, int64_t ib_rows, int64_t ni, int32_t f, int32_t kp,
                               int32_t su, const int32_t* u_row_exp, int32_t si, const int32_t* list_ids,
                               const int32_t* list_pos, const double* bounds, int32_t c, int64_t block,
                               const uint16_t* prefix_b, const double* prefix_norm, const int32_t* prefix_ids,
                               const double* prefix_tile_ceil, int64_t b_pad,
                               const int64_t* q_user, const int64_t* q_perm, const int64_t* q_off, int64_t nq,
                               int32_t k, int32_t* out_ids, double* out_scores, int64_t* out_visited, int32_t options,
                                    void* stream) {
  SIMDEX_CHECK_ARG(users && ub && user_norms && items && ib && item_norms && list_ids && list_pos && bounds &&
                       (block == 0 || (prefix_b && prefix_norm)) && q_user && q_off && out_ids && out_scores &&
                       out_visited,
                   "simdex_query_ws: null pointer");
  SIMDEX_CHECK_ARG(ni >= 1 && f >= 1 && k >= 1 && block >= 0 && c >= 1 && kp % 64 == 0 && kp >= f,
                   "simdex_query_ws: bad sizes");
  SIMDEX_CHECK_ARG(block == 0 || (b_pad % 128 == 0 && b_pad >= (block < ni ? block : ni)),
                   "simdex_query_ws: bad prefix padding");
  const int64_t k_eff = k < ni ? k : ni;
  SIMDEX_CHECK_ARG(k_eff <= kMaxMatmulK && kp <= kMaxKp,
                   "simdex_query_ws: k_eff <= %d and f <= %d required (use simdex_walk)", kMaxMatmulK, kMaxKp);
  if (nq == 0) return SIMDEX_OK;
  Ctx* cx = ctx_or_default(ctx);
  SIMDEX_CHECK_ARG(cx, "simdex_query_ws: no execution context");
  return gemm_topk_ws(users, users32, ub, user_norms, nu, items, items32, ib, item_norms, item_perm, ib_rows, ni, f, kp, su, u_row_exp, si,
                      list_ids, list_pos,
                      bounds, c, block, prefix_b, prefix_norm, prefix_ids, prefix_tile_ceil, b_pad, q_user, q_perm,
                      q_off, nq, k, out_ids,
                      out_scores, out_visited, options, cx, as_stream(stream));
}

extern "C" int simdex_query_ws_opts(const double* users, const float* users32, const uint16_t* ub, const double* user_norms, int64_t nu,
                               const double* items, const float* items32, const uint16_t* ib,
                               const double* item_norms,
                               const int32_t* item_perm, int64_t ib_rows, int64_t ni, int32_t f, int32_t kp,
                               int32_t su, int32_t si, const int32_t* list_ids,
                               const int32_t* list_pos, const double* bounds, int32_t c, int64_t block,
                               const uint16_t* prefix_b, const double* prefix_norm, int64_t b_pad,
                               const int64_t* q_user, const int64_t* q_perm, const int64_t* q_off, int64_t nq,
                               int32_t k, int32_t* out_ids, double* out_scores, int64_t* out_visited, int32_t options,
                                    void* stream) {
  return simdex_query_ws_ctx(nullptr, users, users32, ub, user_norms, nu, items, items32, ib, item_norms, item_perm,
                             ib_rows, ni, f, kp, su, nullptr, si, list_ids, list_pos, bounds, c, block, prefix_b, prefix_norm,
                             nullptr, nullptr, b_pad, q_user, q_perm, q_off, nq, k, out_ids, out_scores, out_visited,
                             options, stream);
}

extern "C" int simdex_query_ws(const double* users, const float* users32, const uint16_t* ub, const double* user_norms, int64_t nu,
                               const double* items, const float* items32, const uint16_t* ib,
                               const double* item_norms,
                               const int32_t* item_perm, int64_t ib_rows, int64_t ni, int32_t f, int32_t kp,
                               int32_t su, int32_t si, const int32_t* list_ids,
                               const int32_t* list_pos, const double* bounds, int32_t c, int64_t block,
                               const uint16_t* prefix_b, const double* prefix_norm, int64_t b_pad,
                               const int64_t* q_user, const int64_t* q_perm, const int64_t* q_off, int64_t nq,
                               int32_t k, int32_t* out_ids, double* out_scores, int64_t* out_visited, void* stream) {
  return simdex_query_ws_opts(users, users32, ub, user_norms, nu, items, items32, ib, item_norms, item_perm, ib_rows,
                              ni, f, kp, su, si, list_ids, list_pos, bounds, c, block, prefix_b, prefix_norm, b_pad,
                              q_user, q_perm, q_off, nq, k, out_ids, out_scores, out_visited, 0, stream);
}
