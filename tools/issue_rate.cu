// MMA issue-cost probe for the kernels' issue pattern: 8 TS MMAs (N=64) per
// "step" whose TMEM A address and smem B descriptor are computed from a TMEM
// base read from shared memory, issued (a) by lane 0 of a warp, (b) the same with
// the base broadcast by __shfl_sync, (c) by the whole warp with elect.sync inside
// the asm.  Reports cycles per MMA.  One CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/issue_rate tools/issue_rate.cu
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2507_04239_b200/csrc/pa_sm100.cuh"

using namespace pa::sm100;

__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

template <int MODE>
__global__ void __launch_bounds__(128, 1) k(int steps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  if (w == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = tid; i < 64 * 1024 / 4; i += 128) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  constexpr uint32_t id = idesc_f16(128, 64, false, true);
  if (w == 1) {
    uint32_t tm = tbase;
    if (MODE == 1) tm = __shfl_sync(0xffffffffu, tm, 0);
    const uint64_t b0 = smem_desc(smem_u32(smem), 8192, 1024, 2);
    long long t0 = clock64();
    if (MODE == 2) {
      for (int s = 0; s < steps; ++s) {
        const uint64_t so = (uint64_t)(((s & 3) * 16384) >> 4);
        const uint32_t ab = tm + 256u + (uint32_t)((s & 1) * 64);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ts_elect(tm + (uint32_t)((s & 1) * 64), ab + kk * 8, b0 + so + kk * 128, id, 1u);
      }
      commit_elect(&bar);
      __syncwarp();
      mbar_wait(&bar, 0);
    } else if (l == 0) {
      for (int s = 0; s < steps; ++s) {
        const uint64_t so = (uint64_t)(((s & 3) * 16384) >> 4);
        const uint32_t ab = tm + 256u + (uint32_t)((s & 1) * 64);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) mma_ts(tm + (uint32_t)((s & 1) * 64), ab + kk * 8, b0 + so + kk * 128, id, 1u);
      }
      tc_commit(&bar);
      mbar_wait(&bar, 0);
    }
    long long t1 = clock64();
    if (l == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tbase);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  const int steps = 1024;
  const char* nm[] = {"lane 0, base from smem", "lane 0, base via shfl", "whole warp, elect in asm"};
  for (int mode = 0; mode < 3; ++mode) {
    auto fn = mode == 0 ? k<0> : (mode == 1 ? k<1> : k<2>);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
    fn<<<148, 128, 70 * 1024>>>(steps, d);
    fn<<<148, 128, 70 * 1024>>>(steps, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    printf("%-28s %.2f cycles per MMA (%s)\n", nm[mode], avg / (steps * 8.0), e ? cudaGetErrorString(e) : "ok");
  }
  return 0;
}
