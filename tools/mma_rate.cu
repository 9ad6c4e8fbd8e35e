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

__device__ __forceinline__ void mma_ts_elect(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc));
}

__global__ void __launch_bounds__(128, 1) rate(int var, int ts, int bmn, int N, int R, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  if (tid < 32) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init(&bar2, 1);
    fence_barrier_init();
  }
  for (int i = tid; i < 96 * 1024 / 4; i += 128) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (var == 0 && tid == 0) {
    // one thread runs the loop (divergent branch)
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
  } else if (var == 1 && tid < 32) {
    // whole warp runs the loop (uniform datapath), one elected lane issues
    const uint32_t id = idesc_f16(128, N, false, bmn != 0);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int i = 0; i < R; i += 4) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t bd = bmn ? smem_desc(b + kk * 2048, 8192, 1024, 2) : smem_desc(b + kk * 32, 16, 1024, 2);
        if (elect_one()) {
          if (ts)
            mma_ts(tm, tm + 256u + (uint32_t)(kk * 8), bd, id, 1u);
          else
            mma_ss(tm, smem_desc(a + kk * 32, 16, 1024, 2), bd, id, 1u);
        }
        __syncwarp();
      }
    }
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  } else if (var == 2 && tid == 0) {
    // one thread, descriptors precomputed, unrolled by 4
    const uint32_t id = idesc_f16(128, N, false, bmn != 0);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    uint64_t bd[4], ad[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      bd[kk] = bmn ? smem_desc(b + kk * 2048, 8192, 1024, 2) : smem_desc(b + kk * 32, 16, 1024, 2);
      ad[kk] = smem_desc(a + kk * 32, 16, 1024, 2);
    }
    long long t0 = clock64();
    for (int i = 0; i < R; i += 4) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (ts)
          mma_ts(tm, tm + 256u + (uint32_t)(kk * 8), bd[kk], id, 1u);
        else
          mma_ss(tm, ad[kk], bd[kk], id, 1u);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  else if (var >= 3 && tid == 0) {
    // one thread, precomputed descriptors, rotating over nacc accumulators
    const int nacc = var == 3 ? 2 : 4;
    const uint32_t id = idesc_f16(128, N, false, bmn != 0);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    uint64_t bd[4], ad[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      bd[kk] = bmn ? smem_desc(b + kk * 2048, 8192, 1024, 2) : smem_desc(b + kk * 32, 16, 1024, 2);
      ad[kk] = smem_desc(a + kk * 32, 16, 1024, 2);
    }
    long long t0 = clock64();
    for (int i = 0; i < R; i += 4) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = tm + (uint32_t)((kk % nacc) * N);
        if (ts)
          mma_ts(acc, tm + 256u + (uint32_t)(kk * 8), bd[kk], id, 1u);
        else
          mma_ss(acc, ad[kk], bd[kk], id, 1u);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  else if (var == 5 && (tid == 0 || tid == 32)) {
    // two issuing warps, separate accumulators
    const uint32_t id = idesc_f16(128, N, false, bmn != 0);
    const uint32_t b = smem_u32(smem + 32768);
    uint64_t bd[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      bd[kk] = bmn ? smem_desc(b + kk * 2048, 8192, 1024, 2) : smem_desc(b + kk * 32, 16, 1024, 2);
    const uint32_t acc = tm + (tid ? 128u : 0u);
    long long t0 = clock64();
    for (int i = 0; i < R / 2; i += 4) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_ts(acc, tm + 256u + (uint32_t)(kk * 8), bd[kk], id, 1u);
    }
    tc_commit(tid ? &bar2 : &bar);
    mbar_wait(tid ? &bar2 : &bar, 0);
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  else if (var >= 6 && tid == 0) {
    // 6: accumulate = 0 ; 7: M = 64 ; 8: kind::f8f6f4 (e4m3, K = 32) ; 9: N=256 baseline
    const int M = var == 7 ? 64 : 128;
    uint32_t id = idesc_f16(M, N, false, bmn != 0);
    if (var == 8) id = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);  // A,B e4m3 (0)
    const uint32_t b = smem_u32(smem + 32768);
    uint64_t bd[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk)
      bd[kk] = smem_desc(b + kk * 32, 16, 1024, 2);
    const int acol = bmn;
    const uint32_t accf = var == 6 ? 0u : 1u;
    long long t0 = clock64();
    for (int i = 0; i < R; i += 4) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (var == 8)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f8f6f4 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
              "r"(tm + 256u + (uint32_t)(kk * 8)), "l"(bd[kk]), "r"(id), "r"(accf));
        else
          mma_ts(tm, tm + (uint32_t)acol + (uint32_t)(kk * 8), bd[kk], id, accf);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  else if (var == 9 && tid < 32) {
    // whole warp, descriptor arithmetic per MMA, elect inside the asm
    const uint32_t id = idesc_f16(128, N, false, false);
    const uint32_t b = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const int kk = i & 3;
      mma_ts_elect(tm, tm + 256u + (uint32_t)(kk * 8), smem_desc(b + (i & 7) * 2048 + kk * 32, 16, 1024, 2), id,
                   i > 0 ? 1u : 0u);
    }
    if (elect_one()) tc_commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = (unsigned long long)(t1 - t0);
  } else if (var == 10 && tid == 0) {
    // single thread, descriptor arithmetic per MMA (like the kernels)
    const uint32_t id = idesc_f16(128, N, false, false);
    const uint32_t b = smem_u32(smem + 32768);
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      const int kk = i & 3;
      mma_ts(tm, tm + 256u + (uint32_t)(kk * 8), smem_desc(b + (i & 7) * 2048 + kk * 32, 16, 1024, 2), id,
             i > 0 ? 1u : 0u);
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

template <int COLS>
__global__ void __launch_bounds__(128, 1) rate2(int N, int R, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  if (tid < 32) tmem_alloc<COLS>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = tid; i < 40 * 1024 / 4; i += 128) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_f16(128, N, false, false);
    const uint32_t b = smem_u32(smem + 16384);
    uint64_t bd[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) bd[kk] = smem_desc(b + kk * 32, 16, 1024, 2);
    long long t0 = clock64();
    for (int i = 0; i < R; i += 4) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_ts(tm, tm + 192u + (uint32_t)(kk * 8), bd[kk], id, 1u);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<COLS>(tm);
}

__global__ void __launch_bounds__(128, 1) rate3(int N, int R, int mode, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, w = tid >> 5;
  if (tid < 32) tmem_alloc<512>(&tbase);
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  for (int i = tid; i < 40 * 1024 / 4; i += 128) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_f16(128, N, false, false);
    const uint32_t b = smem_u32(smem + 16384);
    uint64_t bd[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) bd[kk] = smem_desc(b + kk * 32, 16, 1024, 2);
    long long t0 = clock64();
    for (int i = 0; i < R; i += 4) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) mma_ts(tm, tm + 256u + (uint32_t)(kk * 8), bd[kk], id, 1u);
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = (unsigned long long)(t1 - t0);
  } else if (w >= 1 && mode > 0) {
    // other warps: tcgen05.ld (mode 1) or tcgen05.st (mode 2) traffic on columns [384, 512)
    const uint32_t lane_off = (uint32_t)((w & 3) * 32) << 16;
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = i;
    float acc = 0.f;
    for (int it = 0; it < R / 8; ++it) {
      if (mode == 1) {
        tmem_ld16(tm + 384u + lane_off + (uint32_t)((it & 7) * 16), r);
        tc_wait_ld();
        acc += __uint_as_float(r[it & 15]);
      } else {
        tmem_st16(tm + 384u + lane_off + (uint32_t)((it & 7) * 16), r);
        tc_wait_st();
      }
    }
    if (acc == 12345.f) out[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc<512>(tm);
}

// alternating pattern of the intra-chunk backward: (acc0, A0, B0) / (acc1, A1, B1), K-steps interleaved
__global__ void __launch_bounds__(128, 1) rate4(int mode, int R, unsigned long long* out) {
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
  for (int i = tid; i < 64 * 1024 / 4; i += 128) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  if (tid == 0) {
    const uint32_t id = idesc_bf16(128, 64, false, mode >= 2);
    const uint64_t b0 = smem_desc(smem_u32(smem), mode >= 2 ? 8192 : 16, 1024, 2);
    const uint64_t b1 = smem_desc(smem_u32(smem + 16384), mode >= 2 ? 8192 : 16, 1024, 2);
    long long t0 = clock64();
    for (int i = 0; i < R; i += 8) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (mode == 0 || mode == 2) {
          // two accumulators, two A operands, interleaved
          mma_ts(tm, tm + 384u + kk * 8, b0 + kk * (mode >= 2 ? 128 : 2), id, 1u);
          mma_ts(tm + 64, tm + 416u + kk * 8, b1 + kk * (mode >= 2 ? 128 : 2), id, 1u);
        } else {
          // same accumulator / A for all (baseline)
          mma_ts(tm, tm + 384u + kk * 8, b0 + kk * 2, id, 1u);
          mma_ts(tm, tm + 384u + kk * 8, b0 + kk * 2, id, 1u);
        }
      }
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
  {
    unsigned long long* d4;
    cudaMalloc(&d4, 148 * 8);
    cudaFuncSetAttribute(rate4, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    const char* nm[] = {"two acc/A interleaved, B K-major", "one acc/A, B K-major", "two acc/A interleaved, B MN-major"};
    for (int mode = 0; mode < 3; ++mode) {
      rate4<<<148, 128, 80 * 1024>>>(mode, 8192, d4);
      rate4<<<148, 128, 80 * 1024>>>(mode, 8192, d4);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h[148];
      cudaMemcpy(h, d4, sizeof h, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < 148; ++i) avg += h[i];
      avg /= 148;
      printf("rate4 %-40s N=64: %.2f cyc/MMA (%s)\n", nm[mode], avg / 8192, e ? cudaGetErrorString(e) : "ok");
    }
  }
  return 0;
}
