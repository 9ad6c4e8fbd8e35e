// Throughput probe for tcgen05.mma shapes used by the kernels: one CTA per SM,
// one thread issues R back-to-back MMAs (kind::f16, M = 128), commit once, and
// the CTA reports cycles per MMA.  Modes: A from smem (SS) or TMEM (TS), B
// K-major or MN-major (SW128), N in {16, 64, 128, 256}.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/mma_rate tools/mma_rate.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2507_04239_b200/csrc/pa_sm100.cuh"

using namespace pa::sm100;

__global__ void __launch_bounds__(128, 1) rate(int ts, int bmn, int N, int R, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  if (tid < 32) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = tid; i < 96 * 1024 / 4; i += 128) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_f16(128, N, false, bmn != 0);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const int kk = i & 3;
      uint64_t bd = bmn ? smem_desc(b + kk * 2048, 8192, 1024, 2) : smem_desc(b + kk * 32, 16, 1024, 2);
      if (ts)
        mma_ts(tm, tm + 256u + (uint32_t)(kk * 8), bd, id, 1u);
      else
        mma_ss(tm, smem_desc(a + kk * 32, 16, 1024, 2), bd, id, 1u);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<512>(tm);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int R = 8192;
  for (int ts = 0; ts < 2; ++ts)
    for (int bmn = 0; bmn < 2; ++bmn)
      for (int N : {16, 64, 128, 256}) {
        rate<<<148, 128, 100 * 1024>>>(ts, bmn, N, R, d);
        rate<<<148, 128, 100 * 1024>>>(ts, bmn, N, R, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[148];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        const double cyc = avg / R;
        printf("%s B %s N=%3d : %6.2f cyc/MMA  ideal %5.1f  -> %5.1f%% of 8192 FLOP/clk  %s\n", ts ? "TS" : "SS",
               bmn ? "MN" : "K ", N, cyc, N / 2.0, 100.0 * (N / 2.0) / cyc, e ? cudaGetErrorString(e) : "");
      }
  return 0;
}
