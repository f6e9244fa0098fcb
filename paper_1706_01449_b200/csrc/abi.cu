// C-ABI entry points (include/simdex_b200.h) that are not defined next to
// their kernels, plus the shared error state.
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <vector>
#include <cstdarg>
#include <cstring>

#include "common.cuh"

namespace simdex {

static thread_local char g_err[1024] = "";
static std::atomic<int64_t> g_launches{0};

void count_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ---------------------------------------------------------------------------
// optional per-kernel event timing (simdex_profile_*): events are recorded on
// the launching stream around the named kernels, read back on demand.
// ---------------------------------------------------------------------------
namespace {
struct Pending {
  std::string name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<Pending> g_pending;
std::vector<cudaEvent_t> g_event_pool;  // recycled events: no cudaEventCreate in a timed loop
std::map<std::string, std::pair<double, int64_t>> g_prof_acc;

cudaEvent_t pooled_event() {
  if (!g_event_pool.empty()) {
    cudaEvent_t e = g_event_pool.back();
    g_event_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}
}  // namespace

ProfileScope::ProfileScope(const char* name, cudaStream_t s) : s_(s) {
  if (!g_prof_on) return;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return;
  name_ = name;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    a_ = pooled_event();
    b_ = pooled_event();
  }
  cudaEventRecord(a_, s);
  on_ = true;
}

void ProfileScope::end() {
  if (!on_) return;
  on_ = false;
  cudaEventRecord(b_, s_);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_pending.push_back(Pending{name_, a_, b_});
}

// ---------------------------------------------------------------------------
// execution context
// ---------------------------------------------------------------------------
struct Ctx {
  int device = 0;
  char* arena = nullptr;
  size_t cap = 0;
  cudaStream_t last = nullptr;  // stream of the previous call
  cudaEvent_t done = nullptr;   // end of the previous call on `last`
  bool have_done = false;
  bool busy = false;
  int64_t* host = nullptr;  // pinned statistics slots
  uint64_t arena_gen = 0;   // bumped whenever the arena is (re)allocated
  bool captured = false;    // a CUDA graph holds pointers into the current arena
  std::vector<char*> retired;  // arenas captured into graphs and outgrown since: kept until the context dies
  CtxSetup setup;
};

namespace {
constexpr int kHostSlots = 16;

int ctx_init(Ctx* c, int device) {
  c->device = device;
  SIMDEX_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
  SIMDEX_CUDA(cudaMallocHost(&c->host, kHostSlots * sizeof(int64_t)));
  memset(c->host, 0, kHostSlots * sizeof(int64_t));
  return SIMDEX_OK;
}
}  // namespace

Ctx* ctx_or_default(void* ctx) {
  if (ctx) return reinterpret_cast<Ctx*>(ctx);
  static thread_local std::map<int, Ctx*> per_device;
  int dev = 0;
  cudaGetDevice(&dev);
  auto it = per_device.find(dev);
  if (it != per_device.end()) return it->second;
  Ctx* c = new Ctx();
  if (ctx_init(c, dev) != SIMDEX_OK) {
    delete c;
    return nullptr;
  }
  per_device[dev] = c;
  return c;
}

int64_t* ctx_host_slots(Ctx* c) { return c->host; }
CtxSetup* ctx_setup(Ctx* c) { return &c->setup; }
uint64_t ctx_arena_gen(Ctx* c) { return c->arena_gen; }

Workspace::Workspace(Ctx* c, cudaStream_t s) : c_(c), s_(s) {}

int Workspace::commit() {
  if (!c_) {
    set_error("no execution context");
    return SIMDEX_ECUDA;
  }
  if (c_->busy) {
    set_error("execution context already in use by an enclosing call");
    return SIMDEX_EINVAL;
  }
  // order this call after the context's previous call when the stream changed
  // (not while the stream is being captured into a CUDA graph: a capture may
  // not depend on outside work; the capturing caller orders it, e.g.
  // torch.cuda.graph synchronises first)
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  SIMDEX_CUDA(cudaStreamIsCapturing(s_, &cs));
  capturing_ = cs != cudaStreamCaptureStatusNone;
  if (c_->have_done && c_->last != s_ && !capturing_) SIMDEX_CUDA(cudaStreamWaitEvent(s_, c_->done, 0));
  size_t need = 0;
  for (auto& r : reqs_) need += (r.bytes + 255) & ~size_t(255);
  if (need > c_->cap && capturing_) {
    set_error("execution context: the workspace must be grown (run the call once) before graph capture");
    return SIMDEX_EINVAL;
  }
  if (need > c_->cap) {
    size_t grow = (need + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1);
    // Growth is rare (the first calls of a process) and takes a plain
    // cudaFree + cudaMalloc, which synchronise the device.  An arena regrown
    // through the stream-ordered pool (cudaFreeAsync + cudaMallocAsync, which
    // may stitch the new block from the freed ones) left about one process in
    // eight with a catalogue pass twice as slow for its whole life
    // (tools/full_pass_variation.py; a context whose arena was allocated
    // once was never slow).
    // (an arena a CUDA graph was captured over stays allocated: the graph's
    // kernels hold its addresses and may be replayed after this growth)
    if (c_->arena && c_->captured)
      c_->retired.push_back(c_->arena);
    else if (c_->arena)
      SIMDEX_CUDA(cudaFree(c_->arena));
    c_->captured = false;
    c_->arena = nullptr;
    c_->cap = 0;
    keep_pool_warm();
    SIMDEX_CUDA(cudaMalloc(reinterpret_cast<void**>(&c_->arena), grow));
    c_->cap = grow;
    ++c_->arena_gen;
  }
  size_t off = 0;
  for (auto& r : reqs_) {
    *r.p = c_->arena + off;
    off += (r.bytes + 255) & ~size_t(255);
  }
  c_->busy = true;
  committed_ = true;
  if (capturing_) c_->captured = true;
  // whatever this call leaves in the arena is not a reusable query setup
  // unless the call itself records one (gemm_topk_ws)
  c_->setup.held_token = 0;
  return SIMDEX_OK;
}

Workspace::~Workspace() {
  if (!committed_) return;
  c_->busy = false;
  if (capturing_) return;  // a replayed graph is ordered by its launch stream
  c_->last = s_;
  c_->have_done = cudaEventRecord(c_->done, s_) == cudaSuccess;
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t e, const char* what) {
  set_error("CUDA error %s (%d) at %s", cudaGetErrorString(e), (int)e, what);
  return e == cudaErrorMemoryAllocation ? SIMDEX_ENOMEM : SIMDEX_ECUDA;
}

void keep_pool_warm() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev == done_dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done_dev = dev;
}

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n;
}

int launch_walk(const double*, const double*, const double*, const float*, const float*, int32_t, int64_t,
                const int32_t*, const double*, const int64_t*, const int32_t*, int64_t, int32_t, int64_t,
                const int32_t*, const double*, const int32_t*, int32_t, int32_t*, double*, int64_t*, cudaStream_t);
int launch_pack_f16(const double*, int64_t, int32_t, int32_t, int64_t, int32_t, uint16_t*, double*, cudaStream_t);
int launch_pack_f16_rows(const double*, int64_t, int32_t, int64_t, int32_t, uint16_t*, double*, int32_t*,
                         cudaStream_t);
int launch_build_prefix_ordered(const uint16_t*, const double*, int64_t, int32_t, const double*, int32_t,
                                const double*, const int32_t*, const int32_t*, const double*, int32_t, int64_t,
                                int64_t, uint16_t*, double*, int32_t*, double*, cudaStream_t, int64_t);
int launch_gather_prefix(const uint16_t*, const double*, int64_t, int32_t, const int32_t*, int32_t, int64_t,
                         int64_t, uint16_t*, double*, cudaStream_t);

}  // namespace simdex

using namespace simdex;

extern "C" int simdex_abi_version(void) { return SIMDEX_ABI_VERSION; }

extern "C" const char* simdex_last_error(void) { return g_err; }

extern "C" int64_t simdex_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

extern "C" int simdex_ctx_create(int device, void** out_ctx) {
  SIMDEX_CHECK_ARG(out_ctx, "simdex_ctx_create: null pointer");
  int prev = 0;
  SIMDEX_CUDA(cudaGetDevice(&prev));
  SIMDEX_CUDA(cudaSetDevice(device));
  Ctx* c = new Ctx();
  int rc = ctx_init(c, device);
  cudaSetDevice(prev);
  if (rc != SIMDEX_OK) {
    delete c;
    return rc;
  }
  *out_ctx = c;
  return SIMDEX_OK;
}

extern "C" int simdex_ctx_set_query_token(void* ctx, int64_t token) {
  Ctx* c = ctx_or_default(ctx);
  if (!c) return SIMDEX_ECUDA;
  c->setup.query_token = token;
  return SIMDEX_OK;
}

extern "C" int simdex_ctx_set_full_lists(void* ctx, const uint16_t* full_b, const double* full_norm, int64_t bf_pad) {
  Ctx* c = ctx_or_default(ctx);
  if (!c) return SIMDEX_ECUDA;
  SIMDEX_CHECK_ARG((full_b == nullptr) == (full_norm == nullptr) && bf_pad % 128 == 0 && bf_pad >= 0,
                   "simdex_ctx_set_full_lists: bad arguments");
  c->setup.full_b = full_b;
  c->setup.full_norm = full_norm;
  c->setup.bf_pad = full_b ? bf_pad : 0;
  return SIMDEX_OK;
}

extern "C" int simdex_ctx_destroy(void* ctx) {
  if (!ctx) return SIMDEX_OK;
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  SIMDEX_CHECK_ARG(!c->busy, "simdex_ctx_destroy: context in use");
  int prev = 0;
  SIMDEX_CUDA(cudaGetDevice(&prev));
  SIMDEX_CUDA(cudaSetDevice(c->device));
  if (c->have_done) cudaEventSynchronize(c->done);
  if (c->arena) cudaFree(c->arena);
  for (char* old : c->retired) cudaFree(old);
  if (c->done) cudaEventDestroy(c->done);
  if (c->host) cudaFreeHost(c->host);
  cudaSetDevice(prev);
  delete c;
  return SIMDEX_OK;
}

extern "C" int simdex_ctx_workspace_bytes(void* ctx, int64_t* out_bytes) {
  SIMDEX_CHECK_ARG(out_bytes, "simdex_ctx_workspace_bytes: null pointer");
  Ctx* c = ctx_or_default(ctx);
  SIMDEX_CHECK_ARG(c, "simdex_ctx_workspace_bytes: no context");
  *out_bytes = (int64_t)c->cap;
  return SIMDEX_OK;
}

extern "C" int simdex_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof_on = on != 0;
  return SIMDEX_OK;
}

extern "C" int simdex_profile_read(const char* name, double* total_ms, int64_t* launches) {
  SIMDEX_CHECK_ARG(name && total_ms && launches, "simdex_profile_read: null pointer");
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& p : g_pending) {
    float ms = 0.f;
    SIMDEX_CUDA(cudaEventSynchronize(p.b));
    SIMDEX_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    auto& acc = g_prof_acc[p.name];
    acc.first += ms;
    acc.second += 1;
    g_event_pool.push_back(p.a);
    g_event_pool.push_back(p.b);
  }
  g_pending.clear();
  auto it = g_prof_acc.find(name);
  *total_ms = it == g_prof_acc.end() ? 0.0 : it->second.first;
  *launches = it == g_prof_acc.end() ? 0 : it->second.second;
  return SIMDEX_OK;
}

extern "C" int simdex_profile_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& p : g_pending) {
    cudaEventSynchronize(p.b);
    g_event_pool.push_back(p.a);
    g_event_pool.push_back(p.b);
  }
  g_pending.clear();
  g_prof_acc.clear();
  return SIMDEX_OK;
}

extern "C" int simdex_device_info(int device, int* sms, int* major, int* minor) {
  SIMDEX_CHECK_ARG(sms && major && minor, "simdex_device_info: null pointer");
  SIMDEX_CUDA(cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, device));
  SIMDEX_CUDA(cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, device));
  SIMDEX_CUDA(cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, device));
  return SIMDEX_OK;
}

extern "C" int simdex_topk_exact(const double* users, int64_t nu, const double* items, int64_t ni, int32_t f,
                                 const int64_t* rows, int64_t n_rows, int32_t k, int32_t* out_ids,
                                 double* out_scores, void* stream) {
  SIMDEX_CHECK_ARG(users && items && out_ids && out_scores, "simdex_topk_exact: null pointer");
  SIMDEX_CHECK_ARG(nu >= 1 && ni >= 1 && f >= 1 && k >= 1 && ni < INT32_MAX, "simdex_topk_exact: bad sizes");
  SIMDEX_CHECK_ARG(rows || n_rows == nu, "simdex_topk_exact: n_rows must equal nu without a row list");
  return exact_topk_rows(users, items, ni, f, rows, n_rows, k, out_ids, out_scores, as_stream(stream));
}

namespace simdex {
int launch_max_abs(const double*, int64_t, double*, cudaStream_t);
}

extern "C" int simdex_max_abs(const double* x, int64_t n, double* out, void* stream) {
  SIMDEX_CHECK_ARG(x && out, "simdex_max_abs: null pointer");
  SIMDEX_CHECK_ARG(n >= 0, "simdex_max_abs: bad sizes");
  return launch_max_abs(x, n, out, as_stream(stream));
}

extern "C" int simdex_pack_f16(const double* x, int64_t rows, int32_t f, int32_t scale_exp, int64_t rows_pad,
                                int32_t kp, uint16_t* out_f16, double* out_norms, void* stream) {
  SIMDEX_CHECK_ARG(x && out_f16 && out_norms, "simdex_pack_f16: null pointer");
  SIMDEX_CHECK_ARG(rows >= 1 && f >= 1 && rows_pad >= rows && kp >= f && kp % 64 == 0,
                   "simdex_pack_f16: bad sizes");
  return launch_pack_f16(x, rows, f, scale_exp, rows_pad, kp, out_f16, out_norms, as_stream(stream));
}

extern "C" int simdex_pack_f16_rows(const double* x, int64_t rows, int32_t f, int64_t rows_pad, int32_t kp,
                                    uint16_t* out_f16, double* out_norms, int32_t* out_row_exp, void* stream) {
  SIMDEX_CHECK_ARG(x && out_f16 && out_norms && out_row_exp, "simdex_pack_f16_rows: null pointer");
  SIMDEX_CHECK_ARG(rows >= 1 && f >= 1 && rows_pad >= rows && kp >= f && kp % 64 == 0,
                   "simdex_pack_f16_rows: bad sizes");
  return launch_pack_f16_rows(x, rows, f, rows_pad, kp, out_f16, out_norms, out_row_exp, as_stream(stream));
}

extern "C" int simdex_walk32(const double* users, const double* user_norms, const double* items, const float* users32,
                             const float* items32, int32_t f, int64_t ni, const int32_t* list_ids,
                             const double* bounds, const int64_t* q_user, const int32_t* q_cluster, int64_t nq,
                             int32_t k, int64_t start, const int32_t* warm_ids, const double* warm_scores,
                             const int32_t* warm_count, int32_t no_prune, int32_t* out_ids, double* out_scores,
                             int64_t* out_visited, void* stream) {
  SIMDEX_CHECK_ARG(users && user_norms && items && list_ids && bounds && q_user && q_cluster && out_ids &&
                       out_scores && out_visited,
                   "simdex_walk: null pointer");
  SIMDEX_CHECK_ARG(ni >= 1 && f >= 1 && k >= 1 && nq >= 0 && start >= 0, "simdex_walk: bad sizes");
  SIMDEX_CHECK_ARG(start == 0 || (warm_ids && warm_scores && warm_count), "simdex_walk: warm start needs warm lists");
  if (!(users32 && items32)) users32 = items32 = nullptr;  // both or neither
  return launch_walk(users, user_norms, items, users32, items32, f, ni, list_ids, bounds, q_user, q_cluster, nq, k,
                     start, warm_ids, warm_scores, warm_count, no_prune, out_ids, out_scores, out_visited,
                     as_stream(stream));
}

extern "C" int simdex_walk(const double* users, const double* user_norms, const double* items, int32_t f,
                           int64_t ni, const int32_t* list_ids, const double* bounds, const int64_t* q_user,
                           const int32_t* q_cluster, int64_t nq, int32_t k, int64_t start, const int32_t* warm_ids,
                           const double* warm_scores, const int32_t* warm_count, int32_t no_prune,
                           int32_t* out_ids, double* out_scores, int64_t* out_visited, void* stream) {
  return simdex_walk32(users, user_norms, items, nullptr, nullptr, f, ni, list_ids, bounds, q_user, q_cluster, nq, k,
                       start, warm_ids, warm_scores, warm_count, no_prune, out_ids, out_scores, out_visited, stream);
}

extern "C" int simdex_build_prefix(const uint16_t* ib, const double* i_norm, int64_t ni, int32_t kp,
                                   const int32_t* list_ids, int32_t c, int64_t block, int64_t b_pad,
                                   uint16_t* out_prefix_b, double* out_prefix_norm, void* stream) {
  SIMDEX_CHECK_ARG(ib && i_norm && list_ids && out_prefix_b && out_prefix_norm, "simdex_build_prefix: null pointer");
  SIMDEX_CHECK_ARG(ni >= 1 && c >= 1 && block >= 1 && b_pad >= (block < ni ? block : ni) && kp % 64 == 0,
                   "simdex_build_prefix: bad sizes");
  return launch_gather_prefix(ib, i_norm, ni, kp, list_ids, c, block, b_pad, out_prefix_b, out_prefix_norm,
                              as_stream(stream));
}

extern "C" int simdex_build_prefix_ordered(const uint16_t* ib, const double* i_norm, int64_t ni, int32_t kp,
                                           const double* items, int32_t f, const double* centers,
                                           const int32_t* list_ids, const int32_t* list_pos, const double* bounds,
                                           int32_t c, int64_t block, int64_t b_pad, uint16_t* out_prefix_b,
                                           double* out_prefix_norm, int32_t* out_prefix_ids,
                                           double* out_tile_ceil, void* stream) {
  SIMDEX_CHECK_ARG(ib && i_norm && items && centers && list_ids && list_pos && bounds && out_prefix_b &&
                       out_prefix_norm && out_prefix_ids && out_tile_ceil,
                   "simdex_build_prefix_ordered: null pointer");
  SIMDEX_CHECK_ARG(ni >= 1 && c >= 1 && block >= 1 && f >= 1 && b_pad >= (block < ni ? block : ni) &&
                       b_pad % 128 == 0 && kp % 64 == 0,
                   "simdex_build_prefix_ordered: bad sizes");
  return launch_build_prefix_ordered(ib, i_norm, ni, kp, items, f, centers, list_ids, list_pos, bounds, c, block,
                                     b_pad, out_prefix_b, out_prefix_norm, out_prefix_ids, out_tile_ceil,
                                     as_stream(stream), 0);
}

extern "C" int simdex_build_prefix_hybrid(const uint16_t* ib, const double* i_norm, int64_t ni, int32_t kp,
                                          const double* items, int32_t f, const double* centers,
                                          const int32_t* list_ids, const int32_t* list_pos, const double* bounds,
                                          int32_t c, int64_t block, int64_t b_pad, int64_t head,
                                          uint16_t* out_prefix_b, double* out_prefix_norm, int32_t* out_prefix_ids,
                                          double* out_tile_ceil, void* stream) {
  SIMDEX_CHECK_ARG(ib && i_norm && items && centers && list_ids && list_pos && bounds && out_prefix_b &&
                       out_prefix_norm && out_prefix_ids && out_tile_ceil,
                   "simdex_build_prefix_hybrid: null pointer");
  SIMDEX_CHECK_ARG(ni >= 1 && c >= 1 && block >= 1 && f >= 1 && head >= 0 && b_pad >= (block < ni ? block : ni) &&
                       b_pad % 128 == 0 && kp % 64 == 0,
                   "simdex_build_prefix_hybrid: bad sizes");
  return launch_build_prefix_ordered(ib, i_norm, ni, kp, items, f, centers, list_ids, list_pos, bounds, c, block,
                                     b_pad, out_prefix_b, out_prefix_norm, out_prefix_ids, out_tile_ceil,
                                     as_stream(stream), head);
}

extern "C" int simdex_merge_topk(const int32_t* in_ids, const double* in_scores, int32_t parts, int64_t nu,
                                 int32_t kk, int32_t k_out, int32_t* out_ids, double* out_scores, void* stream) {
  SIMDEX_CHECK_ARG(in_ids && in_scores && out_ids && out_scores, "simdex_merge_topk: null pointer");
  SIMDEX_CHECK_ARG(parts >= 1 && parts <= 32 && nu >= 0 && kk >= 1 && k_out >= 1, "simdex_merge_topk: bad sizes");
  return merge_lists(in_ids, in_scores, parts, nu, kk, k_out, out_ids, out_scores, as_stream(stream));
}
