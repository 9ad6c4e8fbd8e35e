// Latency probe: mbarrier try_wait on an already-completed phase, tcgen05.commit,
// tcgen05.fence, single-thread MMA issue with a completed-barrier wait per step.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o tools/sync_rate tools/sync_rate.cu
#include <cuda_runtime.h>
#include <stdio.h>

#include "../paper_2507_04239_b200/csrc/pa_sm100.cuh"

using namespace pa::sm100;

__global__ void __launch_bounds__(128, 1) k(int mode, int R, unsigned long long* out) {
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  if (tid < 32) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    mbar_arrive(&bar);   // phase 0 complete
    long long t0 = clock64();
    if (mode == 0) {
      for (int i = 0; i < R; ++i) mbar_wait(&bar, 0);
    } else if (mode == 1) {
      for (int i = 0; i < R; ++i) {
        mbar_wait(&bar, 0);
        tc_fence_after();
      }
    } else if (mode == 2) {
      for (int i = 0; i < R; ++i) tc_commit(&bar2);
    } else if (mode == 3) {
      for (int i = 0; i < R; ++i) {
        mbar_try_wait(&bar, 0);
      }
    } else if (mode == 4) {
      int c = 0;
      for (int i = 0; i < R; ++i) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred P;\n\t"
            "mbarrier.test_wait.parity.shared::cta.b64 P, [%1], %2;\n\t"
            "selp.b32 %0, 1, 0, P;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(&bar)), "r"(0u)
            : "memory");
        c += ok;
        if (!ok) break;
      }
      if (c == 7) out[0] = 1;
    } else if (mode == 5) {
      int c = 0;
      for (int i = 0; i < R; ++i) {
        uint32_t ok = mbar_try_wait(&bar, 0) ? 1u : 0u;
        c += ok;
        if (!ok) break;
      }
      if (c == 7) out[0] = 1;
    }
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
  const char* names[] = {"mbar_wait (complete phase)", "mbar_wait + tcgen05.fence::after", "tcgen05.commit",
                         "mbarrier.try_wait only", "test_wait, result consumed", "try_wait, result consumed"};
  for (int mode = 0; mode < 6; ++mode) {
    k<<<148, 128>>>(mode, 1000, d);
    k<<<148, 128>>>(mode, 1000, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    printf("%-36s %.1f cycles each (%s)\n", names[mode], avg / 148 / 1000, e ? cudaGetErrorString(e) : "ok");
  }
  return 0;
}
