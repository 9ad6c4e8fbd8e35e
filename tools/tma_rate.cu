// Tensor-TMA issue probe: one thread per CTA (one CTA per SM) loads 2-D boxes
// (64 x R bf16, SW128) from an L2-resident matrix through a ring of `ns` stages;
// reports cycles per copy.  Compare with tools/l2_stream.cu (1-D bulk copies).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2507_04239_b200/csrc/pa_sm100.cuh"
using namespace pa::sm100;

__global__ void k(const __grid_constant__ CUtensorMap m, int rows_box, int ns, int np, int iters, long long* cyc,
                  int lanes) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[64];
  const int tid = threadIdx.x, w = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < ns * np; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  int pid;
  if (lanes) {   // producers are lanes 0..np-1 of warp 0, converged
    if (w != 0 || (tid & 31) >= np) return;
    pid = tid & 31;
  } else {       // producers are lane 0 of warps 0..np-1
    if ((tid & 31) || w >= np) return;
    pid = w;
  }
  const int tb = rows_box * 128;
  uint64_t* fb = full + pid * ns;
  uint8_t* smw = sm + (size_t)pid * ns * tb;
  long long t0 = clock64();
  for (int i = 0; i < iters + ns; ++i) {
    if (i >= ns) mbar_wait(&fb[(i - ns) % ns], ((i - ns) / ns) & 1);
    if (i < iters) {
      const int st = i % ns;
      mbar_expect_tx(&fb[st], tb);
      tma_load_2d(smw + (size_t)st * tb, &m, &fb[st], 0, (blockIdx.x % 8) * 4096 + ((i * np + pid) * rows_box) % 4096);
    }
  }
  if (pid == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  void* src;
  const size_t rows = 8 * 4096 + 256;
  cudaMalloc(&src, rows * 128);
  cudaMemset(src, 0, rows * 128);
  long long* cyc;
  cudaMalloc(&cyc, 8 * nsm);
  void* fnp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fnp;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct C { int rb, ns, np; };
  const C cs[] = {{64, 8, 1}, {128, 4, 1}, {256, 2, 1}, {64, 4, 2}, {64, 2, 4}, {128, 2, 2}};
  for (int lanes = 0; lanes < 2; ++lanes)
  for (const C& c : cs) {
    CUtensorMap m;
    cuuint64_t dims[2] = {64, rows};
    cuuint64_t str[1] = {128};
    cuuint32_t box[2] = {64, (cuuint32_t)c.rb};
    cuuint32_t es[2] = {1, 1};
    enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int iters = 4000;
    const int smem = c.rb * 128 * c.ns * c.np;
    k<<<nsm, 32 * c.np, smem>>>(m, c.rb, c.ns, c.np, iters, cyc, lanes);
    k<<<nsm, 32 * c.np, smem>>>(m, c.rb, c.ns, c.np, iters, cyc, lanes);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[256];
    cudaMemcpy(h, cyc, 8 * nsm, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < nsm; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%s 2-D TMA box 64 x %3d (%5d B) x %d stages x %d producers: %.0f cycles per copy per producer, %.1f B/clk/SM (%s)\n",
           lanes ? "lanes of one warp:" : "separate warps:   ", c.rb, c.rb * 128, c.ns, c.np, mx / iters, (double)iters * c.rb * 128 * c.np / mx, cudaGetErrorString(e));
  }
  return 0;
}
