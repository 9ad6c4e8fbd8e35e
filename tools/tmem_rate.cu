// TMEM -> register bandwidth probe: W warps per CTA (one CTA per SM) issue
// tcgen05.ld.32x32b.x16 back to back (with or without waiting after each),
// and tcgen05.st the same way.  Reports bytes per cycle per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/tmem_rate tools/tmem_rate.cu
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2507_04239_b200/csrc/pa_sm100.cuh"

using namespace pa::sm100;

__global__ void k(int mode, int R, unsigned long long* out, float* sink) {
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid >> 5;
  if (w == 0) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
  const uint32_t col0 = (uint32_t)((w >> 2) * 64);
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = i;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < R; ++it) {
    const uint32_t a = tm + lane_off + col0 + (uint32_t)((it & 1) * 32);
    if (mode == 0) {
      tmem_ld32(a, r);
      tc_wait_ld();
      acc += __uint_as_float(r[it & 31]);
    } else if (mode == 1) {
      tmem_ld16(a, r);
      tmem_ld16(a + 16, r + 16);
      tmem_ld16(a + 32, r);   // more in flight before the wait
      tmem_ld16(a + 48, r + 16);
      tc_wait_ld();
      acc += __uint_as_float(r[it & 31]);
    } else {
      tmem_st16(a, r);
      tmem_st16(a + 16, r + 16);
      tc_wait_st();
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  if (acc == 1234.5f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long* d;
  float* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4);
  const char* nm[] = {"ld x32 + wait", "ld 4x x16 + wait", "st 2x x16 + wait"};
  const int R = 4096;
  for (int mode = 0; mode < 3; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      k<<<148, warps * 32>>>(mode, R, d, sink);
      k<<<148, warps * 32>>>(mode, R, d, sink);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      const double bytes_per_it = (mode == 1 ? 8192.0 : 4096.0) * warps;   // per CTA per iteration
      printf("%-18s warps %2d: %.1f cycles/iter, %.0f B/cycle/SM (%s)\n", nm[mode], warps, avg / R,
             bytes_per_it / (avg / R), e ? cudaGetErrorString(e) : "ok");
    }
  return 0;
}
