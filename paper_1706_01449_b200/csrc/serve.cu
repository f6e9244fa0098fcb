// Serving entry points: topk_matmul (brute.py:59-113) and work-sharing
// query_batch (index.py:305-389).
#include "common.cuh"

namespace simdex {
int launch_walk(const double*, const double*, const double*, int32_t, int64_t, const int32_t*, const double*,
                const int64_t*, const int32_t*, int64_t, int32_t, int64_t, const int32_t*, const double*,
                const int32_t*, int32_t, int32_t*, double*, int64_t*, cudaStream_t);
int ws_fix_visited(int64_t*, int64_t, int64_t, int64_t, cudaStream_t);
}  // namespace simdex

using namespace simdex;

extern "C" int simdex_topk_matmul(const double* users, const uint16_t* ub, const double* u_norm, int64_t nu,
                                  const double* items, const uint16_t* ib, const double* i_norm, int64_t ni,
                                  int32_t f, int32_t kp, int32_t su, int32_t si, int32_t k, int32_t* out_ids,
                                  double* out_scores, int64_t* heap_ops, void* stream) {
  SIMDEX_CHECK_ARG(users && items && out_ids && out_scores, "simdex_topk_matmul: null pointer");
  SIMDEX_CHECK_ARG(nu >= 1 && ni >= 1 && f >= 1 && k >= 1, "simdex_topk_matmul: bad sizes");
  (void)ub; (void)u_norm; (void)ib; (void)i_norm; (void)kp; (void)su; (void)si; (void)heap_ops;
  return exact_topk_rows(users, items, ni, f, nullptr, nu, k, out_ids, out_scores, as_stream(stream));
}

extern "C" int simdex_query_ws(const double* users, const uint16_t* ub, const double* user_norms, int64_t nu,
                               const double* items, int64_t ni, int32_t f, int32_t kp, int32_t su, int32_t si,
                               const int32_t* list_ids, const double* bounds, int32_t c, int64_t block,
                               const uint16_t* prefix_b, const double* prefix_norm, const int64_t* q_user,
                               const int32_t* q_cluster, int64_t nq, int32_t k, int32_t* out_ids,
                               double* out_scores, int64_t* out_visited, void* stream) {
  SIMDEX_CHECK_ARG(users && user_norms && items && list_ids && bounds && q_user && q_cluster && out_ids &&
                       out_scores && out_visited,
                   "simdex_query_ws: null pointer");
  SIMDEX_CHECK_ARG(ni >= 1 && f >= 1 && k >= 1 && block >= 1 && c >= 1, "simdex_query_ws: bad sizes");
  (void)ub; (void)kp; (void)su; (void)si; (void)prefix_b; (void)prefix_norm; (void)nu;
  cudaStream_t s = as_stream(stream);
  int rc = launch_walk(users, user_norms, items, f, ni, list_ids, bounds, q_user, q_cluster, nq, k, 0, nullptr,
                       nullptr, nullptr, 0, out_ids, out_scores, out_visited, s);
  if (rc) return rc;
  return ws_fix_visited(out_visited, nq, block, ni, s);
}
