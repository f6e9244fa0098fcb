// Microbenchmark: TMEM read bandwidth (tcgen05.ld) per SM and legacy
// mma.sync (HMMA m16n8k16 f16 -> f32) throughput per SM on sm_100a.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o ubench_tmem tools/ubench_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ uint32_t ld_x(uint32_t taddr);

template <>
__device__ __forceinline__ uint32_t ld_x<32>(uint32_t taddr) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) x ^= r[i];
  return x;
}

// 16x256b.x8: 16 lanes x 256 bits x 8 -> 32 regs per thread
__device__ __forceinline__ uint32_t ld_16x256(uint32_t taddr) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x256b.x8.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) x ^= r[i];
  return x;
}

// 32x32b.x16 with .pack::16b: 16 pairs of 16-bit columns -> 16 regs (32 columns)
__device__ __forceinline__ uint32_t ld_pack16(uint32_t taddr) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  uint32_t x = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) x ^= r[i];
  return x;
}

template <int MODE>
__global__ void tmem_bw(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = slot;
  const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
  const int colgrp = warp >> 2;
  uint32_t x = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t col = (uint32_t)(((it + colgrp * 3) & 15) * 32);
    if (MODE == 0) x ^= ld_x<32>(base + lane_off + col);
    if (MODE == 1) x ^= ld_16x256(base + lane_off + col);
    if (MODE == 2) x ^= ld_pack16(base + lane_off + col);
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = x;
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(512) : "memory");
}

__global__ void hmma_tp(int iters, unsigned long long* cyc, float* sink) {
  float d[4][4] = {};
  uint32_t a[4] = {0x3c003c00u ^ threadIdx.x, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u};
  uint32_t b[2] = {0x3c003c00u, 0x3c003c00u ^ threadIdx.x};
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(d[j][0]), "+f"(d[j][1]), "+f"(d[j][2]), "+f"(d[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  float s = 0;
  for (int j = 0; j < 4; ++j)
    for (int i = 0; i < 4; ++i) s += d[j][i];
  sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  const int iters = 4096;
  for (int mode = 0; mode < 3; ++mode) {
    for (int warps : {4, 8, 16}) {
      for (int grid : {1, 148}) {
        auto k = mode == 0 ? tmem_bw<0> : mode == 1 ? tmem_bw<1> : tmem_bw<2>;
        k<<<grid, warps * 32>>>(iters, cyc, sink);
        k<<<grid, warps * 32>>>(iters, cyc, sink);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        // bytes per warp-load: 32x32b.x32 = 4 KB; 16x256b.x8 = 32 regs x 32 thr x 4 B = 4 KB; pack16 = 2 KB of regs (4 KB of 16-bit... reads 32 cols x 32 lanes x 32 bit)
        const double bytes = (double)warps * iters * 4096.0;
        printf("tmem mode %d (%s) warps %2d grid %3d: %s %.1f cyc/iter/warp, %.1f B/cyc/SM (4 KB TMEM per ld)\n", mode,
               mode == 0 ? "32x32b.x32" : mode == 1 ? "16x256b.x8" : "32x32b.x32.pack16", warps, grid,
               cudaGetErrorString(e), (double)c / iters, bytes / c);
      }
    }
  }
  for (int warps : {4, 8, 16}) {
    hmma_tp<<<148, warps * 32>>>(iters, cyc, (float*)sink);
    hmma_tp<<<148, warps * 32>>>(iters, cyc, (float*)sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long c = 0;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    const double flops = (double)warps * iters * 4 * 2 * 16 * 8 * 16;
    printf("hmma m16n8k16 f32acc warps %2d: %s %.1f flop/cyc/SM (x148x1.965e9 = %.0f TF)\n", warps,
           cudaGetErrorString(e), flops / c, flops / c * 148 * 1.965e9 / 1e12);
  }
  return 0;
}
