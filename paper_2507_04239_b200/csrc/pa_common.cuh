// Shared device helpers and the problem geometry used by every kernel.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace pa {

// Per-launch geometry.  Streams s = (batch, head) pairs; tokens of stream s
// live at rows ((bi*t + m)*h + hi) of a [b, t, h, x] tensor when bth=1, or at
// rows (s*t + m) of a stream-major [ns, t, x] tensor when bth=0.
struct Geo {
  int b, t, h, d, e, E1;  // E1 = e + 1 (value columns + the score-sum column)
  int p, c, n, D, ns;     // degree, chunk, chunks, features, streams
  float scale;
  int normalize, gated, bth;
  // Sequence-parallel partition (tensor-core path): this launch holds global
  // chunks [k0, k0 + n) of a sequence of ng chunks; prefix = 1 when a state
  // flows in from earlier chunks.  Chunk-state buffers hold nsl = n + 1 slots
  // per stream: slot j is the state before local chunk j (slot 0 = prefix).
  int k0, ng, prefix, nsl;
  // PA_FLAG_DETERMINISTIC: one MMA issuer per accumulator (fixed summation order)
  int det;
  // tokens of the caller's sequence; t > treal when a partial last chunk runs on a
  // zero-padded copy (tensor-core path)
  int treal;
  int dtype;   // pa_dtype of q, k, v
  int keysum;  // PA_FLAG_KEY_SUM: states carry the key-sum column even without normalize
};

__host__ __device__ __forceinline__ size_t rowid(const Geo& g, int s, int m) {
  if (!g.bth) return (size_t)s * g.t + m;
  int bi = s / g.h, hi = s - bi * g.h;
  return ((size_t)bi * g.t + m) * g.h + hi;
}

template <typename T> __device__ __forceinline__ float to_f(T x);
template <> __device__ __forceinline__ float to_f<float>(float x) { return x; }
template <> __device__ __forceinline__ float to_f<double>(double x) { return (float)x; }
template <> __device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 x) { return __bfloat162float(x); }
template <> __device__ __forceinline__ float to_f<__half>(__half x) { return __half2float(x); }

template <typename T> __device__ __forceinline__ T from_f(float x);
template <> __device__ __forceinline__ float from_f<float>(float x) { return x; }
template <> __device__ __forceinline__ double from_f<double>(float x) { return x; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ __half from_f<__half>(float x) { return __float2half_rn(x); }

template <typename A>
__device__ __forceinline__ A ipow(A x, int p) {
  A r = x;
  for (int i = 1; i < p; ++i) r *= x;
  return p == 0 ? A(1) : r;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum; every thread gets the result.  Needs blockDim.x % 32 == 0.
__device__ __forceinline__ float block_sum(float v, float* red /*[32]*/) {
  v = warp_sum(v);
  int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float r = (l < nw) ? red[l] : 0.f;
  return warp_sum(r);
}

// Per-stage device timing (CUDA events on the launching stream), enabled by
// pa_profile_enable(1).  Scope object: records start on construction, end on
// destruction.
struct StageTimer {
  StageTimer(const char* name, cudaStream_t st);
  ~StageTimer();
  const char* name;
  cudaStream_t st;
  cudaEvent_t a;
};

// error plumbing shared by the host side
void set_error(const std::string& msg);
int cuda_check(const char* what);
void count_launch(int n = 1);

}  // namespace pa
