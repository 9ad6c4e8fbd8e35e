// L2 -> shared memory streaming probe: every CTA (one per SM) bulk-copies tiles
// of `tb` bytes from a 512 KB region (L2-resident after the first pass) through a
// ring of `ns` stages per producer; `np` producer warps (lane 0 of each issues
// its own ring in parallel).  Reports bytes/clk/SM and the chip total, and the
// issue cost per copy.
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2507_04239_b200/csrc/pa_sm100.cuh"
using namespace pa::sm100;

__global__ void k_stream(const uint8_t* src, size_t reg, int tb, int ns, int iters, int np, int mode,
                         long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[64];
  const int tid = threadIdx.x, w = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < ns * np; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  if ((tid & 31) != 0 || w >= np) return;
  const uint8_t* base = src + (size_t)(blockIdx.x / 8) * reg;
  uint64_t* fb = full + w * ns;
  uint8_t* smw = sm + (size_t)w * ns * tb;
  const int ntile = (int)(reg / tb);
  long long t0 = clock64();
  for (int i = 0; i < iters + ns; ++i) {
    if (i >= ns) {
      if (mode == 1) {
        while (!mbar_try_wait(&fb[(i - ns) % ns], ((i - ns) / ns) & 1)) {
        }
      } else {
        mbar_wait(&fb[(i - ns) % ns], ((i - ns) / ns) & 1);
      }
    }
    if (i < iters) {
      const int st = i % ns;
      mbar_expect_tx(&fb[st], tb);
      bulk_load(smw + (size_t)st * tb, base + (size_t)((i * np + w) % ntile) * tb, tb, &fb[st]);
    }
  }
  long long t1 = clock64();
  if (w == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const size_t reg = 512 * 1024;
  uint8_t* src;
  cudaMalloc(&src, reg * nsm);
  cudaMemset(src, 1, reg * nsm);
  long long* cyc;
  cudaMalloc(&cyc, 8 * nsm);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Cfg { int tb, ns, np; };
  const Cfg cfgs[] = {{8192, 8, 1}, {8192, 4, 2}, {8192, 4, 4}, {8192, 2, 8}, {8192, 6, 4}, {16384, 4, 2},
                      {16384, 2, 4}, {32768, 4, 1}, {65536, 2, 1}, {4096, 8, 4}, {2048, 8, 8}};
  for (int mode = 0; mode < 2; ++mode)
    for (const Cfg& c : cfgs) {
      const int iters = (int)((64ull << 20) / c.tb / 8 / c.np);
      const int smem = c.tb * c.ns * c.np;
      k_stream<<<nsm, 32 * c.np, smem>>>(src, reg, c.tb, c.ns, iters, c.np, mode, cyc);
      k_stream<<<nsm, 32 * c.np, smem>>>(src, reg, c.tb, c.ns, iters, c.np, mode, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[256];
      cudaMemcpy(h, cyc, 8 * nsm, cudaMemcpyDeviceToHost);
      double mx = 0;
      for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
      const double bytes = (double)iters * c.tb * c.np;
      printf("%s tile %6d B x %d stages x %d producers (%4d KB in flight): %.1f B/clk/SM, chip %.2f TB/s, %.0f cyc/copy/producer (%s)\n",
             mode ? "spin-wait" : "mbar_wait", c.tb, c.ns, c.np, smem / 1024, bytes / mx,
             bytes / mx * nsm * 1.965e9 / 1e12, mx / iters, cudaGetErrorString(e));
    }
  return 0;
}
