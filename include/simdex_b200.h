/*
 * simdex_b200.h -- C ABI of the B200-native exact top-K serving path
 * (SimDex, arXiv 1706.01449; reference package `mipserve`).
 *
 * The reference is pure Python (numpy); it has no FFI.  Each entry point below
 * replaces one numpy call site / function of the reference's hot path and is
 * what a ctypes / cffi binding of that function binds.
 *
 * Conventions
 *   - every pointer is a DEVICE pointer on the current CUDA device unless the
 *     comment says "host";  matrices are row-major and dense;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default);
 *     all work is enqueued on it, nothing synchronises the host unless the
 *     comment says so.  The serving calls (simdex_topk_matmul_ctx,
 *     simdex_query_ws*) allocate nothing per call (their scratch lives in an
 *     execution context, see simdex_ctx_create) and keep every count on the
 *     device, so they can run ahead of the GPU and be captured in a CUDA
 *     graph.  Host-synchronising entry points: simdex_topk_matmul (legacy
 *     form: reads two item norms to pick the early exit), simdex_topk_exact
 *     with k_eff > 4096, simdex_kmeans_seed's degenerate branch (host RNG),
 *     simdex_profile_read;
 *   - factor matrices are float64 [rows, f] like the reference's FactorMatrix
 *     (model_io.py:37-48);  item ids / list positions are int32 (|I| < 2^31);
 *     user ids are int64;
 *   - returns SIMDEX_OK (0) or a negative SIMDEX_E* code; the message is in
 *     simdex_last_error() (thread-local).  Argument validation that raises
 *     ValueError in the reference is done by the Python host mirror first;
 *     the library re-checks shapes and pointers and returns SIMDEX_EINVAL.
 *   - ordering of every top-K result: score descending, item id ascending
 *     (index.py:158-163).  k_eff = min(k, |I|) (brute.py:49, index.py:204).
 */
#ifndef SIMDEX_B200_H
#define SIMDEX_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIMDEX_ABI_VERSION 1

#if defined(__GNUC__)
#define SIMDEX_API __attribute__((visibility("default")))
#else
#define SIMDEX_API
#endif

enum {
  SIMDEX_OK = 0,
  SIMDEX_EINVAL = -1,
  SIMDEX_ECUDA = -2,
  SIMDEX_ENOMEM = -3,
  SIMDEX_EUNSUPPORTED = -4
};

SIMDEX_API int simdex_abi_version(void);
SIMDEX_API const char* simdex_last_error(void);
/* Number of kernels this library has launched in the process (monotone). */
SIMDEX_API int64_t simdex_launch_count(void);
/* Optional per-kernel timing: with profiling on, the library records a CUDA
 * event pair on the launching stream around its main kernels (gemm_topk,
 * finalize, walk, kmeans_assign, ...); simdex_profile_read(name, ...) returns
 * the accumulated milliseconds and launch count for that kernel name (it
 * synchronises on the recorded events). */
SIMDEX_API int simdex_profile_enable(int on);
SIMDEX_API int simdex_profile_read(const char* name, double* total_ms, int64_t* launches);
SIMDEX_API int simdex_profile_reset(void);
/* Execution contexts.  A context owns a device workspace arena (grown on
 * demand with cudaFree + cudaMalloc -- a growing call synchronises the
 * device, which happens only in a process's first calls -- and reused by
 * every later call) and pinned host
 * statistic slots; calls that take `ctx` carve their scratch from it instead
 * of allocating.  ctx == NULL selects the calling thread's default context
 * for the current device (what the legacy entry points use).  A context
 * serves one call at a time; successive calls on different streams are
 * ordered through an event.  Replaces the per-call numpy temporaries of the
 * reference (brute.py:86-107, index.py:351-389) with one resident arena. */
SIMDEX_API int simdex_ctx_create(int device, void** out_ctx);
SIMDEX_API int simdex_ctx_destroy(void* ctx);
/* Declare that the next simdex_query_ws_ctx (or simdex_kmeans_assign) call on `ctx` (NULL: this thread's
 * default context) serves the query set identified by `token` (nonzero,
 * unique for the lifetime of that query set and of the operands it is served
 * with; 0 = none); the call consumes the token.  A call that finds its setup
 * for the same token, inputs and arena still in the context's workspace (no
 * other call has used the context since) skips it: the grouping of the
 * queries into 128-row units, the packed query rows and their bands, and the
 * prefix and catalogue norms (index.py:346-357 done once per query set). */
SIMDEX_API int simdex_ctx_set_query_token(void* ctx, int64_t token);
/* Hand the next simdex_query_ws_ctx call on `ctx` (NULL: this thread's
 * default) every cluster's whole list as a packed operand in list order
 * (simdex_build_prefix with block = n: fp16 [c, bf_pad, kp] and float64 norms
 * [c, bf_pad], bf_pad % 128 == 0); consumed by that call.  With it, the users
 * that go on past B are grouped by cluster and scan their own cluster's list
 * from B in ceiling order, stopping on the list ceilings (Algorithm 1's own
 * bound, index.py:225-227) instead of scanning the norm-sorted catalogue; the
 * prefix top-K joins their candidates.  Same results, less work.  NULL
 * pointers: the norm-sorted catalogue pass. */
SIMDEX_API int simdex_ctx_set_full_lists(void* ctx, const uint16_t* full_b, const double* full_norm, int64_t bf_pad);
/* current arena size of `ctx` in bytes (host output) */
SIMDEX_API int simdex_ctx_workspace_bytes(void* ctx, int64_t* out_bytes);

/* sm count / compute capability of `device` (host outputs). */
SIMDEX_API int simdex_device_info(int device, int* sm_count, int* cc_major, int* cc_minor);

/* ------------------------------------------------------------------------
 * Brute force (brute.py)
 * ---------------------------------------------------------------------- */

/* brute.py:43-56 topk_naive: exact float64 score of every (row, item) pair and
 * the full (score desc, id asc) ordering, truncated to k_eff.
 * rows: optional int64[n_rows] subset of user rows (NULL: all nu rows, n_rows = nu).
 * out_ids int32[n_rows, k_eff], out_scores float64[n_rows, k_eff]. */
SIMDEX_API int simdex_topk_exact(const double* users, int64_t nu, const double* items, int64_t ni, int32_t f,
                      const int64_t* rows, int64_t n_rows, int32_t k,
                      int32_t* out_ids, double* out_scores, void* stream);

/* max |x[i]| over n values into *out (device float64); picks the packing scale. */
SIMDEX_API int simdex_max_abs(const double* x, int64_t n, double* out, void* stream);

/* Operand packing for the tensor-core path: fp16 copy of x * 2^scale_exp,
 * zero padded to [rows_pad, kp] (kp = 64*ceil(f/64), rows_pad >= rows), and
 * float64 row norms of the UNSCALED rows.  Replaces the fp64->operand
 * conversion implicit in brute.py:93 (dgemm on FactorMatrix values). */
SIMDEX_API int simdex_pack_f16(const double* x, int64_t rows, int32_t f, int32_t scale_exp,
                     int64_t rows_pad, int32_t kp, uint16_t* out_f16, double* out_norms, void* stream);

/* simdex_pack_f16 with one exact power-of-two scale PER ROW (the user
 * operand): out_row_exp int32[rows] receives e_r with max|x_r| 2^e_r in
 * [1, 2) (0 for an all-zero row).  A small-norm row then keeps fp16's full
 * relative precision, so its certified band stays as narrow as a large row's
 * (with one matrix-wide scale its entries sink into fp16 subnormals and the
 * band widens toward the exact fallback).  Pass out_row_exp as u_row_exp to
 * simdex_topk_matmul_ctx / simdex_query_ws_ctx. */
SIMDEX_API int simdex_pack_f16_rows(const double* x, int64_t rows, int32_t f, int64_t rows_pad, int32_t kp,
                     uint16_t* out_f16, double* out_norms, int32_t* out_row_exp, void* stream);

/* brute.py:59-113 topk_matmul: users x items product on tcgen05 tensor cores
 * (single-pass fp16 operands, fp32 accumulation in TMEM) fused with a
 * certified running top-K, then exact float64 rescoring of the surviving
 * candidates.  Results equal simdex_topk_exact.
 *   ub/ib: packed operands from simdex_pack_f16 (same kp, scale exps su/si);
 *   u_norm/i_norm: float64 norms of the unscaled rows;
 *   heap_ops: optional int64[nu]: per user count of tile scores above the
 *   running K-th at the time the tile is merged (brute.py:95-97; tile order
 *   differs from the reference, the count is analogous, not bit-equal).
 *   users32 / items32 (nullable): exact float32 copies for the rescoring reads;
 *   item_perm (nullable): the item operand ib / i_norm is in this row order
 *   (e.g. simdex_norm_order), ib has ib_rows rows (0: 256*ceil(ni/256)).
 * Requires k_eff <= 256; larger k goes through simdex_topk_exact. */
SIMDEX_API int simdex_topk_matmul(const double* users, const float* users32, const uint16_t* ub, const double* u_norm, int64_t nu,
                       const double* items, const float* items32, const uint16_t* ib, const double* i_norm,
                       const int32_t* item_perm, int64_t ib_rows, int64_t ni,
                       int32_t f, int32_t kp, int32_t su, int32_t si, int32_t k,
                       int32_t* out_ids, double* out_scores, int64_t* heap_ops, void* stream);

/* simdex_topk_matmul in an execution context with option bits:
 *   SIMDEX_MM_NORM_EXIT  item_perm is a descending-norm order and the pass
 *     stops streaming a unit once no later item can enter any row's
 *     certified band (Cauchy-Schwarz); pays on skewed norms;
 *   SIMDEX_MM_NORM_AUTO  decide NORM_EXIT from the operand (reads the largest
 *     and the median norm: one host synchronisation).
 * u_row_exp (nullable): per-row scale exponents of ub (simdex_pack_f16_rows),
 * overriding su.  Without NORM_AUTO the call never synchronises the host. */
#define SIMDEX_MM_NORM_EXIT 2
#define SIMDEX_MM_NORM_AUTO 4
SIMDEX_API int simdex_topk_matmul_ctx(void* ctx, const double* users, const float* users32, const uint16_t* ub,
                       const double* u_norm, int64_t nu, const double* items, const float* items32,
                       const uint16_t* ib, const double* i_norm, const int32_t* item_perm, int64_t ib_rows,
                       int64_t ni, int32_t f, int32_t kp, int32_t su, const int32_t* u_row_exp, int32_t si, int32_t k,
                       int32_t* out_ids, double* out_scores, int64_t* heap_ops, int32_t options, void* stream);

/* ------------------------------------------------------------------------
 * Clustering (clustering.py)
 *
 * The k-means entry points take the points as float64 (`points`) or, when
 * the caller has verified the values are exactly representable (BASELINE
 * inputs are float32 upcast), as the float32 copy `points32` (non-NULL wins):
 * the arithmetic is float64 either way, the float32 copy halves the bytes.
 * ---------------------------------------------------------------------- */

/* float32 copy of x[n]; *inexact (device int32) = 1 if any value changed. */
SIMDEX_API int simdex_to_f32(const double* x, int64_t n, float* out, int32_t* inexact, void* stream);

/* clustering.py:105-122 _plusplus_seeds on device.  The host draws the RNG
 * stream exactly as the reference: first = rng.integers(0, n), then one
 * rng.random() per further seed (numpy's choice(n, p) == searchsorted(cdf, u,
 * 'right')).  uniforms: float64[k-1] (device).  Writes out_rows int64[k] (the
 * chosen point ids) and out_centers float64[k, f].  If a pass finds a
 * non-positive D^2 total (fewer distinct points than seeds,
 * clustering.py:113-117), *out_degenerate_pass (device int32) receives that
 * pass index and the remaining rows are left for the host; else -1. */
SIMDEX_API int simdex_kmeans_seed(const double* points, const float* points32, int64_t n, int32_t f, int32_t k,
                       int64_t first,
                       const double* uniforms, int64_t* out_rows, double* out_centers,
                       int32_t* out_degenerate_pass, void* stream);

/* clustering.py:96-102 + argmin (:164, :176): squared L2 distances to every
 * center as ||p||^2 + ||c||^2 - 2 p.c clipped at 0, first minimum wins.
 * prev_assign (nullable) is compared to count changed rows.
 * out_assign int64[n], out_d2 float64[n] (distance to the assigned center),
 * out_changed int64[1], out_objective float64[1] = sum(out_d2).
 * Runs on the thread's default context; a token set with
 * simdex_ctx_set_query_token(NULL, t) (t unique to one run over the same,
 * unchanged points, e.g. the Lloyd loop of clustering.py:160-190) lets
 * consecutive calls reuse the point side of the product (squared norms,
 * packed operand, bands) while nothing else has used that context. */
SIMDEX_API int simdex_kmeans_assign(const double* points, const float* points32, int64_t n, int32_t f,
                         const double* centers, int32_t c,
                         const int64_t* prev_assign, int64_t* out_assign, double* out_d2,
                         int64_t* out_changed, double* out_objective, void* stream);

/* clustering.py:168-172 (+ members, :185): users sorted by (cluster, id)
 * into out_members int64[n] with out_offsets int64[c+1]; out_counts int64[c];
 * centers[c] <- mean of its members for every non-empty cluster (fixed
 * summation order: deterministic). */
SIMDEX_API int simdex_kmeans_update(const double* points, const float* points32, int64_t n, int32_t f,
                         const int64_t* assign, int32_t c,
                         double* centers, int64_t* out_counts, int64_t* out_members, int64_t* out_offsets,
                         void* stream);

/* clustering.py:65-93 compute_max_angles: theta_b[c] = max over members of
 * 2*atan2(|x-y|, |x+y|) on unit vectors; zero-norm member or center -> pi;
 * empty cluster -> 0.  out_theta float64[c]. */
SIMDEX_API int simdex_max_angles(const double* users, int64_t n, int32_t f, const double* centers, int32_t c,
                      const int64_t* assign, double* out_theta, void* stream);

/* ------------------------------------------------------------------------
 * Index build (index.py:90-155)
 * ---------------------------------------------------------------------- */

/* index.py:129-155 build_index: item norms, per (cluster, item) half-angle
 * theta_ic (zero-norm item / zero center -> pi/2, index.py:103-116), Eq. 2
 * ceiling (index.py:119-121), and per-cluster sort by (ceiling desc, id asc)
 * (index.py:124-126) -- a device merge sort.
 * out_item_norms float64[ni], out_list_ids int32[c, ni], out_bounds float64[c, ni],
 * out_list_pos int32[c, ni] (nullable): position of item i in cluster c's list. */
SIMDEX_API int simdex_build_index(const double* items, int64_t ni, int32_t f, const double* centers,
                       const double* theta_b, int32_t c, double* out_item_norms,
                       int32_t* out_list_ids, double* out_bounds, int32_t* out_list_pos, void* stream);

/* Items by (norm desc, id asc): out_perm int32[n].  The brute-force pass
 * streams the catalogue in this order so each row's threshold rises early and
 * low-norm tiles are rejected by the norm bound (simdex_topk_matmul item_perm). */
SIMDEX_API int simdex_norm_order(const double* norms, int64_t n, int32_t* out_perm, void* stream);

/* Inverse list permutation: out_pos[c, list_ids[c, j]] = j (int32[c, ni]). */
SIMDEX_API int simdex_list_positions(const int32_t* list_ids, int32_t c, int64_t ni, int32_t* out_pos, void* stream);

/* ------------------------------------------------------------------------
 * Index walk (index.py:185-389)
 * ---------------------------------------------------------------------- */

/* index.py:185-268 _walk / query_user, one query per entry:
 *   q_user int64[nq] user row, q_cluster int32[nq] its cluster (list row);
 *   start: first list position (0, or the work-sharing prefix B);
 *   warm_ids/warm_scores [nq, k_eff] + warm_count int32[nq]: the running
 *   top-K entering at `start` (nullable when start == 0);
 *   no_prune != 0 scans the whole list (the per-pair baseline, brute.py:116-130).
 * Exact Algorithm 1 semantics: first k_eff positions scored unconditionally,
 * stop at the first later position j with kth > bounds[j]*||u|| (strict).
 * out_ids int32[nq, k_eff], out_scores float64[nq, k_eff], out_visited int64[nq]. */
SIMDEX_API int simdex_walk(const double* users, const double* user_norms, const double* items, int32_t f, int64_t ni,
                const int32_t* list_ids, const double* bounds,
                const int64_t* q_user, const int32_t* q_cluster, int64_t nq, int32_t k, int64_t start,
                const int32_t* warm_ids, const double* warm_scores, const int32_t* warm_count,
                int32_t no_prune, int32_t* out_ids, double* out_scores, int64_t* out_visited, void* stream);

/* simdex_walk reading exact float32 copies of users / items (both or
 * neither; NULL: the float64 values): half the bytes per scored item, the
 * arithmetic float64 either way (every float32 value is exact in float64).
 * Scoring is coalesced: 8-lane groups read one contiguous item row each.
 * A k_eff whose top-K does not fit a warp's shared memory (k beyond ~16k)
 * is answered by the exact scan, visited from Algorithm 1's closed form
 * (start == 0 only). */
SIMDEX_API int simdex_walk32(const double* users, const double* user_norms, const double* items,
                const float* users32, const float* items32, int32_t f, int64_t ni,
                const int32_t* list_ids, const double* bounds,
                const int64_t* q_user, const int32_t* q_cluster, int64_t nq, int32_t k, int64_t start,
                const int32_t* warm_ids, const double* warm_scores, const int32_t* warm_count,
                int32_t no_prune, int32_t* out_ids, double* out_scores, int64_t* out_visited, void* stream);

/* index.py:305-389 query_batch with work sharing: every cluster's first B
 * list items scored for all its queried users on tcgen05 (prefix GEMM fused
 * with the certified top-K, as simdex_topk_matmul), then the walk continues
 * from B only for users whose K-th does not beat the ceiling at B.
 * Queries are grouped by cluster (simdex_group_queries): cluster j's queries
 * are q_user[q_off[j] .. q_off[j+1]); grouped query i is written to output
 * row q_perm[i] (q_perm NULL: row i).  prefix_b / prefix_norm are the
 * per-cluster prefix operands from simdex_build_prefix ([c, b_pad, kp]).
 * Users whose K-th does not beat the ceiling at B are finished by a second
 * certified tensor-core pass over the whole catalogue (ib / item_norms, the
 * simdex_pack_f16 operand of the items); their Algorithm 1 stop position
 * then follows in closed form from the exact top-K (list_pos = inverse of
 * list_ids, from simdex_build_index).
 * out_visited follows the reference: n if B >= n, else max(B, walk visited).
 * block == 0: no work sharing (query_batch(work_sharing=False)): every query
 * takes the full-list pass and out_visited is Algorithm 1's stop position
 * from position 0, exactly simdex_walk's; prefix_b / prefix_norm may be NULL.
 * Requires k_eff <= 256 and f <= 256 (else use simdex_walk). */
SIMDEX_API int simdex_query_ws(const double* users, const float* users32, const uint16_t* ub, const double* user_norms, int64_t nu,
                    const double* items, const float* items32, const uint16_t* ib, const double* item_norms,
                    const int32_t* item_perm, int64_t ib_rows, int64_t ni,
                    int32_t f, int32_t kp, int32_t su, int32_t si,
                    const int32_t* list_ids, const int32_t* list_pos, const double* bounds, int32_t c, int64_t block,
                    const uint16_t* prefix_b, const double* prefix_norm, int64_t b_pad,
                    const int64_t* q_user, const int64_t* q_perm, const int64_t* q_off, int64_t nq, int32_t k,
                    int32_t* out_ids, double* out_scores, int64_t* out_visited, void* stream);

/* simdex_query_ws with option bits (simdex_query_ws == options 0):
 *   SIMDEX_WS_PREFIX_EXIT  the prefix pass ends a 128-query unit once every
 *     query's certified K-th lower bound exceeds ||u|| x the list ceiling at
 *     the next 128-item tile (Algorithm 1's own stop bound, index.py:225-227);
 *     results are identical.  It pays when walks are short against B (the
 *     optimizer's estimate, optimizer.py:117-145, well below B) and costs a
 *     few percent otherwise. */
#define SIMDEX_WS_PREFIX_EXIT 1
SIMDEX_API int simdex_query_ws_opts(const double* users, const float* users32, const uint16_t* ub, const double* user_norms, int64_t nu,
                    const double* items, const float* items32, const uint16_t* ib, const double* item_norms,
                    const int32_t* item_perm, int64_t ib_rows, int64_t ni,
                    int32_t f, int32_t kp, int32_t su, int32_t si,
                    const int32_t* list_ids, const int32_t* list_pos, const double* bounds, int32_t c, int64_t block,
                    const uint16_t* prefix_b, const double* prefix_norm, int64_t b_pad,
                    const int64_t* q_user, const int64_t* q_perm, const int64_t* q_off, int64_t nq, int32_t k,
                    int32_t* out_ids, double* out_scores, int64_t* out_visited, int32_t options, void* stream);

/* simdex_query_ws_opts in an execution context (NULL: the thread default);
 * u_row_exp (nullable): per-row scale exponents of ub (simdex_pack_f16_rows);
 * prefix_ids / prefix_tile_ceil (nullable, both or neither): a prefix operand
 * from simdex_build_prefix_ordered (rows in its own order; ids resolve them,
 * tile_ceil bounds the early exit). */
SIMDEX_API int simdex_query_ws_ctx(void* ctx, const double* users, const float* users32, const uint16_t* ub,
                    const double* user_norms, int64_t nu,
                    const double* items, const float* items32, const uint16_t* ib, const double* item_norms,
                    const int32_t* item_perm, int64_t ib_rows, int64_t ni,
                    int32_t f, int32_t kp, int32_t su, const int32_t* u_row_exp, int32_t si,
                    const int32_t* list_ids, const int32_t* list_pos, const double* bounds, int32_t c, int64_t block,
                    const uint16_t* prefix_b, const double* prefix_norm, const int32_t* prefix_ids,
                    const double* prefix_tile_ceil, int64_t b_pad,
                    const int64_t* q_user, const int64_t* q_perm, const int64_t* q_off, int64_t nq, int32_t k,
                    int32_t* out_ids, double* out_scores, int64_t* out_visited, int32_t options, void* stream);

/* Host-side statistics of this thread's last simdex_query_ws call (host
 * int64[5]): queries, queries that went on past B (second pass over the
 * catalogue), B' = min(B, n), n, f.  Lets a caller count the algorithmic
 * tensor work 2*f*(nq*B' + n_cont*n) of the call.  The continuing count is
 * copied to the host asynchronously: read it after the call's stream has
 * synchronised. */
SIMDEX_API int simdex_ws_stats(int64_t* out5);

/* Rows of this thread's last simdex_topk_matmul* / simdex_query_ws* call whose
 * certified band outgrew the candidate buffer and were answered by the exact
 * float64 fallback (host int64; read after the call's stream synchronised). */
SIMDEX_API int simdex_fallback_rows(int64_t* out);

/* (user, item) pairs the tensor-core launches of this thread's last
 * simdex_topk_matmul* / simdex_query_ws* call actually multiplied (valid rows
 * x valid items of every tile issued; the early exits skip tiles): host
 * int64[2] = [brute-force or prefix launch, catalogue launch (0 if none)].
 * Read after the call's stream synchronised.  The roofline's "executed" flop
 * count is 2 f x these pairs. */
SIMDEX_API int simdex_executed_pairs(int64_t* out2);

/* The same counts for the last serving call made on execution context `ctx`
 * (NULL: this thread's default), so a caller running several calls on their
 * own contexts can add them up: host int64[4] = [queries that went on past B
 * (simdex_query_ws_ctx), band-overflow rows, pairs of the first launch, pairs
 * of the catalogue launch].  Read after the calls' streams synchronised. */
SIMDEX_API int simdex_ctx_stats(void* ctx, int64_t* out4);

/* Group queries by their cluster (index.py:346-348), stable in query order:
 * out_q_user int64[nq] grouped user rows, out_perm int64[nq] original query
 * position of each grouped entry, out_off int64[c+1] cluster offsets. */
SIMDEX_API int simdex_group_queries(const int64_t* q_user, int64_t nq, const int64_t* assign, int32_t c,
                         int64_t* out_q_user, int64_t* out_perm, int64_t* out_off, void* stream);

/* Diagnostic: raw fp32 accumulators of the tcgen05 product of two packed
 * operands (simdex_pack_f16 layout), out float[nu, ni].  Used by the tests to
 * validate the TMA/UMMA descriptors against a float reference. */
SIMDEX_API int simdex_gemm_debug(const uint16_t* ub, int64_t nu, const uint16_t* ib, int64_t ni, int32_t f,
                      int32_t kp, float* out, void* stream);

/* Work-sharing operands: for every cluster the first min(B, ni) list items,
 * gathered in list order into fp16 [c, b_pad, kp] (b_pad = 128*ceil(B'/128))
 * plus their float64 norms [c, b_pad]; the re-layout that makes the prefix
 * product a dense TMA-fed GEMM (index.py:351-357). */
SIMDEX_API int simdex_build_prefix(const uint16_t* ib, const double* i_norm, int64_t ni, int32_t kp,
                        const int32_t* list_ids, int32_t c, int64_t block, int64_t b_pad,
                        uint16_t* out_prefix_b, double* out_prefix_norm, void* stream);

/* simdex_build_prefix with each cluster's B' items in "likely score" order:
 * sorted by the centroid's float64 score centers[j] . items[i] (desc, id asc)
 * instead of list order, so the cluster's users meet their best items first
 * and their certified thresholds rise at once.  The prefix top-K and visited
 * do not depend on the order in which the prefix is scored (index.py:351-387).
 *   items float64 [ni, f], centers float64 [c, f], list_pos = inverse lists;
 *   out_prefix_ids int32 [c, b_pad]: item id of each operand row (-1 padding);
 *   out_tile_ceil float64 [c, b_pad/128]: per 128-row tile, the largest list
 *   ceiling at or after it (the prefix early-exit bound). */
SIMDEX_API int simdex_build_prefix_ordered(const uint16_t* ib, const double* i_norm, int64_t ni, int32_t kp,
                        const double* items, int32_t f, const double* centers,
                        const int32_t* list_ids, const int32_t* list_pos, const double* bounds, int32_t c,
                        int64_t block, int64_t b_pad, uint16_t* out_prefix_b, double* out_prefix_norm,
                        int32_t* out_prefix_ids, double* out_tile_ceil, void* stream);
/* The same with a hybrid order: each cluster's `head` prefix items with the
 * best centroid scores first, then the rest of the prefix in list (ceiling)
 * order, so that out_tile_ceil falls like the list's ceilings past the head
 * and the early exit (SIMDEX_WS_PREFIX_EXIT) can end a warp inside the
 * prefix (index.py:225-227).  head = 0: simdex_build_prefix_ordered. */
SIMDEX_API int simdex_build_prefix_hybrid(const uint16_t* ib, const double* i_norm, int64_t ni, int32_t kp,
                        const double* items, int32_t f, const double* centers,
                        const int32_t* list_ids, const int32_t* list_pos, const double* bounds, int32_t c,
                        int64_t block, int64_t b_pad, int64_t head, uint16_t* out_prefix_b, double* out_prefix_norm,
                        int32_t* out_prefix_ids, double* out_tile_ceil, void* stream);

/* ------------------------------------------------------------------------
 * Catalog sharding (no reference counterpart)
 * ---------------------------------------------------------------------- */

/* Merge `parts` partial top-K lists per user into one: in_ids/in_scores
 * [parts, nu, kk] (ids already global), output [nu, k_out] by
 * (score desc, id asc). */
SIMDEX_API int simdex_merge_topk(const int32_t* in_ids, const double* in_scores, int32_t parts, int64_t nu,
                      int32_t kk, int32_t k_out, int32_t* out_ids, double* out_scores, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SIMDEX_B200_H */
