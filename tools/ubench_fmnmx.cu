// Issue rate of the 3-input float max (the gemm_topk epilogue's chunk-max tree)
// against FFMA and 2-input max, per SM: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
// tools/ubench_fmnmx.cu -o build/ubench_fmnmx && build/ubench_fmnmx
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) k(float* out, int iters, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + threadIdx.x * 0.001f + i;
  const float b = seed * 0.5f, c = seed * 0.25f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) a[i] = fmaf(a[i], b, c);
        if (OP == 1) a[i] = fmaxf(a[i] + 0.f, b);  // (the add keeps the chain from folding)
        if (OP == 2) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(b + it), "f"(c + r));
        if (OP == 3) asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(b + it));
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int OP>
void run(const char* name, int per_iter) {
  int dev = 0, sms = 0, khz = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
  const int iters = 4000;
  for (int ctas = 1; ctas <= 8; ctas *= 2) {
    k<OP><<<sms * ctas, 256>>>(out, 10, 1.f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<OP><<<sms * ctas, 256>>>(out, iters, 1.f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_instr = (double)ctas * 8 * iters * 16 * 8 * per_iter;  // per SM
    const double cycles = ms * 1e-3 * khz * 1e3;
    printf("%-10s %d warps/SM: %.2f warp-instructions / cycle / SM\n", name, ctas * 8, warp_instr / cycles);
  }
  cudaFree(out);
}

int main() {
  run<0>("FFMA", 1);
  run<3>("max2", 1);
  run<2>("max3", 1);
  return 0;
}
