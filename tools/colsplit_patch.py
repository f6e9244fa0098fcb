p='paper_1706_01449_b200/csrc/gemm_topk.cu'
s=open(p).read()
def rep(old,new,cnt=1):
    global s
    assert s.count(old)==cnt, (old[:90], s.count(old))
    s=s.replace(old,new)
rep('''constexpr int kEpiWarps = 4 * kMTiles;
constexpr int kThreads = 32 * (2 + kEpiWarps);''','''constexpr int kEpiWarps = 4 * kMTiles;
constexpr int kThreads = 32 * (2 + kEpiWarps);
#ifndef SIMDEX_COLSPLIT
#define SIMDEX_COLSPLIT 1
#endif
template <int KT>
constexpr int epi_warps() {
  return (SIMDEX_COLSPLIT && kMTiles == 1 && KT >= 1 && KT <= 16) ? 8 : kEpiWarps;
}
template <int KT>
constexpr int gemm_threads() {
  return 32 * (2 + epi_warps<KT>());
}
constexpr size_t kTshBytes = 2 * 128 * 8;''')
rep('''  float* debug_out;
  int64_t debug_ld;''','''  float* debug_out;
  int64_t debug_ld;
  int64_t half_stride;''')
rep('''template <int KT, int EXM>
__global__ void __launch_bounds__(kThreads, kCtasPerSm)
    gemm_topk_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const TopkParams p) {''','''template <int KT, int EXM>
__global__ void __launch_bounds__(gemm_threads<KT>(), kCtasPerSm)
    gemm_topk_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const TopkParams p) {
  constexpr int EW = epi_warps<KT>();
  constexpr bool CS = EW == 8 && kMTiles == 1;
  constexpr int CPW = CS ? 2 : kTileN / 32;
  constexpr int LDC = CS ? 1 : 2;''')
rep('''  volatile long long* wdone = reinterpret_cast<volatile long long*>(bars) + 40;  // [8] (unit << 32) | tile after which a warp is done''','''  volatile long long* wdone = reinterpret_cast<volatile long long*>(bars) + 40;  // [8] (unit << 32) | tile after which a warp is done
  volatile unsigned long long* tsh = reinterpret_cast<volatile unsigned long long*>(reinterpret_cast<uint8_t*>(bars) + 512);''')
rep('''      mbar_init(t_empty + b, kEpiWarps);''','''      mbar_init(t_empty + b, EW);''')
rep('''          for (int w = 0; stop && w < kEpiWarps; ++w) {''','''          for (int w = 0; stop && w < EW; ++w) {''')
rep('''  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();''','''  if (warp == 1) tmem_alloc(tmem_slot, kTmemCols);
  if (CS)
    for (int i = threadIdx.x; i < 256; i += blockDim.x) tsh[i] = ~0ull;
  tc_fence_before();
  __syncthreads();''')
rep('''    const int ew = warp - 2;
    const int h = ew >> 2;   // M tile of this warp
    const int q = warp & 3;  // TMEM lane quarter this warp may access''','''    const int ew = warp - 2;
    const int h = CS ? 0 : ew >> 2;
    const int hf = CS ? ew >> 2 : 0;
    const int q = warp & 3;  // TMEM lane quarter this warp may access''')
rep('''      const int64_t srow = un.s_row0 + row_local;  // this (row, catalogue segment)'s state''','''      const int64_t srow = un.s_row0 + hf * p.half_stride + row_local;''')
rep('''        bool released = false;
        if (h < ntile_a && !(EX && done)) {
          const int tile_valid = min(kTileN, un.n_items - t * kTileN);
          // two chunks of 32 columns per TMEM wait; once the whole tile is in
          // registers the accumulator buffer goes back to the MMA warp
          constexpr int LDC = 2;
#pragma unroll
          for (int cg = 0; cg < kTileN / 32; cg += LDC) {
            if (cg * 32 >= tile_valid) break;''','''        bool released = false;
        if constexpr (CS) {
          const int ti = q * 32 + lane;
          tsh[hf * 128 + ti] = ((unsigned long long)(unsigned)u << 32) | __float_as_uint(T);
          const unsigned long long o = tsh[(hf ^ 1) * 128 + ti];
          if ((unsigned)(o >> 32) == (unsigned)u && !flags) T = fmaxf(T, __uint_as_float((unsigned)o));
        }
        if (h < ntile_a && !(EX && done)) {
          const int tile_valid = min(kTileN, un.n_items - t * kTileN);
#pragma unroll
          for (int ci = 0; ci < CPW; ci += LDC) {
            const int cg = hf * CPW + ci;
            if (cg * 32 >= tile_valid) break;''')
rep('''            if (cg + LDC >= kTileN / 32) {''','''            if (ci + LDC >= CPW) {''')
rep('''                if (t == 0 && ch == 0 && nvalid >= 32 &&''','''                if (t == 0 && ch == hf * CPW && nvalid >= 32 &&''')
rep('''  const size_t fixed = 1024 + kMTiles * (size_t)g->kb * kSlab + 512;''','''  const size_t fixed = 1024 + kMTiles * (size_t)g->kb * kSlab + 512 + kTshBytes;''')
rep('''  kern<<<grid, kThreads, g.smem, s>>>(ma, mb, p);''','''  kern<<<grid, gemm_threads<KT>(), g.smem, s>>>(ma, mb, p);''')
rep('''struct RowState {
  int32_t *cid = nullptr, *cnt = nullptr, *flags = nullptr;
  float *lo = nullptr, *hi = nullptr, *rowT = nullptr;
  int cap = 0;
  void add(Workspace& ws, int64_t rows, int k_eff) {
    cap = cap_for(k_eff);
    ws.add(&cid, (size_t)rows * cap);
    ws.add(&hi, (size_t)rows * cap);
    ws.add(&lo, kt_for(k_eff) > 0 ? 1 : (size_t)rows * cap);
    ws.add(&cnt, rows);
    ws.add(&flags, rows);
    ws.add(&rowT, rows);
  }
};''','''bool colsplit_for(int k_eff) {
  const int kt = kt_for(k_eff);
  return SIMDEX_COLSPLIT && kMTiles == 1 && kt >= 1 && kt <= 16;
}
struct RowState {
  int32_t *cid = nullptr, *cnt = nullptr, *flags = nullptr;
  float *lo = nullptr, *hi = nullptr, *rowT = nullptr;
  int cap = 0;
  int64_t rows = 0, half_stride = 0;
  void add(Workspace& ws, int64_t rows_, int k_eff) {
    cap = cap_for(k_eff);
    rows = rows_;
    const int64_t tot = colsplit_for(k_eff) ? 2 * rows : rows;
    half_stride = colsplit_for(k_eff) ? rows : 0;
    ws.add(&cid, (size_t)tot * cap);
    ws.add(&hi, (size_t)tot * cap);
    ws.add(&lo, kt_for(k_eff) > 0 ? 1 : (size_t)tot * cap);
    ws.add(&cnt, tot);
    ws.add(&flags, tot);
    ws.add(&rowT, tot);
  }
};
__global__ void merge_halves_kernel(int64_t rows, int64_t hs, int cap, int32_t* __restrict__ cid,
                                    float* __restrict__ chi, int32_t* __restrict__ cnt, int32_t* __restrict__ flags,
                                    float* __restrict__ rowT) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = r + hs;
    const int cq = min(max(cnt[q], 0), cap);
    int c = min(max(cnt[r], 0), cap);
    const float T = fmaxf(rowT[r], rowT[q]);
    int fl = flags[r] | flags[q];
    for (int e = 0; e < cq && !fl; ++e) {
      const float h = chi[q * cap + e];
      if (h >= T) {
        if (c >= cap) { fl = 1; break; }
        chi[r * cap + c] = h;
        cid[r * cap + c] = cid[q * cap + e];
        ++c;
      }
    }
    cnt[r] = c;
    flags[r] = fl;
    rowT[r] = T;
  }
}
int merge_halves(const RowState& st, int64_t rows, cudaStream_t s) {
  if (!st.half_stride) return SIMDEX_OK;
  merge_halves_kernel<<<(unsigned)std::min<int64_t>(ceil_div(rows, 256), 4 * sm_count()), 256, 0, s>>>(
      rows, st.half_stride, st.cap, st.cid, st.hi, st.cnt, st.flags, st.rowT);
  SIMDEX_LAUNCH_CHECK("merge_halves");
  return SIMDEX_OK;
}''')
rep('''  p.row_T_out = st.rowT;''','''  p.row_T_out = st.rowT;
  p.half_stride = st.half_stride;''')
rep('''  if ((rc = launch_gemm(ma, mb, p, g, grid, "gemm_topk", s))) return rc;''','''  if ((rc = launch_gemm(ma, mb, p, g, grid, "gemm_topk", s))) return rc;
  if ((rc = merge_halves(st, nu_pad, s))) return rc;''')
rep('''    if ((rc = launch_gemm(ma, mb, p, g, grid, "gemm_topk_prefix", s))) return rc;''','''    if ((rc = launch_gemm(ma, mb, p, g, grid, "gemm_topk_prefix", s))) return rc;
    if ((rc = merge_halves(st, rows_max, s))) return rc;''')
rep('''  if ((rc = launch_gemm(ma2, mb2, p2, g, grid, "gemm_topk_full", s))) return rc;''','''  if ((rc = launch_gemm(ma2, mb2, p2, g, grid, "gemm_topk_full", s))) return rc;
  if ((rc = merge_halves(st, rows_max, s))) return rc;''')
rep('''  if ((rc = launch_gemm(ma, mb, tp, g, grid, "gemm_assign", s))) return rc;''','''  if ((rc = launch_gemm(ma, mb, tp, g, grid, "gemm_assign", s))) return rc;
  if ((rc = merge_halves(st, nu_pad, s))) return rc;''')
open(p,'w').write(s)
