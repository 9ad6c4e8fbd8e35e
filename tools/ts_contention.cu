// TS-MMA (A in TMEM) throughput under concurrent TMEM stores: one (or two) warps
// issue M=128 N=64 K=16 kind::f16 MMAs with A from TMEM, while `nst` other warps
// store to other TMEM columns with tcgen05.st (as A-generating warps do).
// Reports cycles per MMA and the TMEM store rate.  One CTA per SM.
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2507_04239_b200/csrc/pa_sm100.cuh"

using namespace pa::sm100;

__global__ void __launch_bounds__(384, 1) k(int steps, int nst, int two, int mn, unsigned long long* out,
                                            unsigned long long* stcnt) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar[2];
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  if (w == 0) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    stop = 0;
    fence_barrier_init();
  }
  for (int i = tid; i < 64 * 1024 / 4; i += 384) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  const uint32_t id = mn ? idesc_f16(128, 64, false, true) : idesc_f16(128, 64, false, false);
  if (w == 0 || (two && w == 1)) {
    const uint64_t b0 = mn ? smem_desc(smem_u32(smem), 8192, 1024, 2) : smem_desc(smem_u32(smem), 16, 1024, 2);
    long long t0 = clock64();
    for (int s = w; s < steps; s += (two ? 2 : 1)) {
      const uint64_t so = (uint64_t)(((s & 3) * 8192) >> 4);
      const uint32_t acc = tm + (uint32_t)((s & 1) * 64);
      const uint32_t ab = tm + 128u + (uint32_t)((s & 3) * 32);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_ts_w(acc, ab + kk * 8, b0 + so + (mn ? kk * 128 : kk * 2), id, 1u);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_ts_w(acc, ab + kk * 8, b0 + so + (mn ? kk * 128 : kk * 2), id, 1u);
    }
    tc_commit_w(&bar[w]);
    mbar_wait_w(&bar[w], 0);
    long long t1 = clock64();
    if (l == 0) out[blockIdx.x * 2 + w] = (unsigned long long)(t1 - t0);
    if (w == 0 && l == 0) stop = 1;
  } else if (w >= 2 && w < 2 + nst) {
    // TMEM stores to columns [256, 512) in this warp's lane quadrant
    const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
    uint32_t v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = i;
    unsigned long long n = 0;
    while (!stop) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st16(tm + lane_off + 256u + (uint32_t)(((w >> 2) * 64 + c * 16) & 255), v);
      tc_wait_st();
      n += 4;
    }
    if (l == 0) atomicAdd(stcnt + blockIdx.x, n);
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tbase);
}

int main() {
  unsigned long long *d, *c;
  cudaMalloc(&d, 148 * 16);
  cudaMalloc(&c, 148 * 8);
  const int steps = 2048;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  for (int mn = 0; mn < 2; ++mn)
    for (int two = 0; two < 2; ++two)
      for (int nst : {0, 4, 8}) {
        cudaMemset(c, 0, 148 * 8);
        k<<<148, 384, 70 * 1024>>>(steps, nst, two, mn, d, c);
        cudaMemset(c, 0, 148 * 8);
        k<<<148, 384, 70 * 1024>>>(steps, nst, two, mn, d, c);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[296], hc[148];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        cudaMemcpy(hc, c, sizeof hc, cudaMemcpyDeviceToHost);
        double avg = 0, st = 0;
        for (int i = 0; i < 148; ++i) {
          avg += h[2 * i];
          st += hc[i];
        }
        avg /= 148;
        st /= 148;
        // each x16 store = 32 lanes x 16 columns x 4 B = 2 KB
        printf("B %s, %s issuer(s), %d storing warps: %.2f cycles per MMA, TMEM stores %.0f B/clk (%s)\n",
               mn ? "MN-major" : "K-major ", two ? "two" : "one", nst, avg / (steps * 8.0), st * 2048.0 / avg,
               e ? cudaGetErrorString(e) : "ok");
      }
  return 0;
}
