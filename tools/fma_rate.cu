// FP32 pipe probe: FFMA (3-register) vs FFMA2 (f32x2) throughput per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fma_rate tools/fma_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t fma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

template <int MODE>
__global__ void k(float* out, int iters, float x0, float y0) {
  float a[16], b = x0 + threadIdx.x, c = y0;
  uint64_t p[8];
  for (int i = 0; i < 16; ++i) a[i] = b + i;
  for (int i = 0; i < 8; ++i) p[i] = ((uint64_t)__float_as_uint(a[2 * i]) << 32) | __float_as_uint(a[2 * i + 1]);
  const uint64_t bb = ((uint64_t)__float_as_uint(b) << 32) | __float_as_uint(c);
  const uint64_t cc = ((uint64_t)__float_as_uint(c) << 32) | __float_as_uint(b);
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], b, c);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) p[i] = fma2(p[i], bb, cc);
    }
  }
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  for (int i = 0; i < 8; ++i) s += __uint_as_float((uint32_t)p[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int mode = 0; mode < 2; ++mode) {
    for (int warps : {4, 8, 16, 32}) {
      for (int r = 0; r < 2; ++r) {
        cudaEventRecord(e0);
        if (mode == 0) k<0><<<148, warps * 32>>>(d, iters, 1.0001f, 0.9999f);
        else k<1><<<148, warps * 32>>>(d, iters, 1.0001f, 0.9999f);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r) {
          const double fmas = 148.0 * warps * 32 * iters * 16;
          printf("%s warps/SM %2d: %.1f TFMA/s = %.1f FMA/clk/SM at 1.965 GHz\n", mode ? "FFMA2" : "FFMA ", warps,
                 fmas / ms / 1e9, fmas / (ms * 1e-3) / 148 / 1.965e9);
        }
      }
    }
  }
  return 0;
}
