// Log-space (stabilised) attention form of power attention: SURVEY §8f row 4,
// reference attention.py:273-309 (use_log_space branch, 289-305).
//
// Per stream (b, h) and query row i, over keys j <= i:
//   ls_ij   = p * log(|sigma q_i . k_j| + eps) + log G_ij,  G_ij = prod_{u=j+1..i} g_u
//   m_i     = max_j ls_ij                      (row max)
//   w_ij    = exp(ls_ij - m_i)
//   shifted = sum_j w_ij,  numer = sum_j w_ij v_j
//   y_i     = numer / shifted        (normalize)   or numer * exp(m_i)   (not)
//   rowsum  = shifted * exp(m_i)
// Zero gates are exact (gate_decay_matrix attention.py:196-205 has no log
// tricks): a pair whose decay window (j, i] holds a zero gate gets weight 0,
// tracked through the index of the last zero gate instead of log(0).
//
// One warp per query row, eight rows per CTA.  The CTA first builds, in shared
// memory, the inclusive prefix L_u = sum_{v<=u, g_v>0} log g_v and the last-
// zero index Z_u for u <= its last row (block scan over the stream's gates),
// so log G_ij = L_i - L_j when Z_i <= j.  Pass 1: lanes stride over keys and
// reduce the row max.  Pass 2: lanes compute 32 weights into shared memory,
// then each lane accumulates value columns lane, lane+32, ... (coalesced v
// rows).  Work is O(t^2 (d + e)) per stream on CUDA cores: this is the
// numerically stabilised form for moderate t, not the throughput path (which
// is the tensor-core chunked pipeline).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "../../include/power_attention_b200.h"
#include "pa_common.cuh"

namespace pa {
namespace {

constexpr int kRowsPerCta = 8;
constexpr int kThreads = 32 * kRowsPerCta;
constexpr int kMaxE = 128;

template <typename T>
__global__ void __launch_bounds__(kThreads) k_logspace_attention(
    int t, int h, int d, int e, int p, T scale, T eps, int normalize, int gated,
    const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
    const T* __restrict__ log_g, T* __restrict__ y, T* __restrict__ rowsum) {
  extern __shared__ unsigned char smem_raw[];
  const int stream = blockIdx.y;  // b * h + head
  const int bi = stream / h, hi = stream % h;
  const int row0 = blockIdx.x * kRowsPerCta;
  const int last = min(row0 + kRowsPerCta, t) - 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // shared layout: L[t] (double), Z[t] (int), qrow[8][d] (T), w[8][32] (T)
  double* L = reinterpret_cast<double*>(smem_raw);
  int* Z = reinterpret_cast<int*>(L + t);
  T* qs = reinterpret_cast<T*>(Z + ((t + 1) & ~1));
  T* ws = qs + kRowsPerCta * d;
  __shared__ double part_l[kThreads];
  __shared__ int part_z[kThreads];

  const int64_t tok_stride = (int64_t)h;  // [b, t, h, x]: token step in rows
  auto gate_at = [&](int u) -> T { return log_g[((int64_t)bi * t + u) * tok_stride + hi]; };

  // ---- block scan of log gates over [0, last] ----
  const int n = last + 1;
  const int per = (n + kThreads - 1) / kThreads;
  const int s0 = threadIdx.x * per, s1 = min(s0 + per, n);
  double acc = 0.0;
  int z = -1;
  if (gated) {
    for (int u = s0; u < s1; ++u) {
      T lg = gate_at(u);
      if (isinf(lg) && lg < T(0)) z = u;
      else acc += (double)lg;
    }
  }
  part_l[threadIdx.x] = acc;
  part_z[threadIdx.x] = z;
  __syncthreads();
  if (threadIdx.x == 0) {
    double run = 0.0;
    int rz = -1;
    for (int i = 0; i < kThreads; ++i) {
      double a = part_l[i];
      int zz = part_z[i];
      part_l[i] = run;
      part_z[i] = rz;
      run += a;
      rz = max(rz, zz);
    }
  }
  __syncthreads();
  {
    double run = part_l[threadIdx.x];
    int rz = part_z[threadIdx.x];
    for (int u = s0; u < s1; ++u) {
      if (gated) {
        T lg = gate_at(u);
        if (isinf(lg) && lg < T(0)) rz = u;
        else run += (double)lg;
      }
      L[u] = run;
      Z[u] = rz;
    }
  }
  // ---- this warp's query row into shared memory (pre-scaled) ----
  const int i = row0 + warp;
  T* qrow = qs + warp * d;
  if (i < t) {
    const T* qi = q + (((int64_t)bi * t + i) * h + hi) * d;
    for (int c = lane; c < d; c += 32) qrow[c] = scale * qi[c];
  }
  __syncthreads();
  if (i >= t) return;

  const double Li = L[i];
  const int Zi = Z[i];
  const int j_lo = max(Zi, 0);  // keys before the last zero gate carry weight 0
  const T pf = T(p);
  auto logscore = [&](int j) -> T {
    const T* kj = k + (((int64_t)bi * t + j) * h + hi) * d;
    T s = T(0);
    for (int c = 0; c < d; ++c) s += qrow[c] * kj[c];
    T ls = pf * log(fabs(s) + eps);
    if (gated) ls += T(Li - L[j]);
    return ls;
  };

  // pass 1: row max
  T m = -INFINITY;
  for (int j = j_lo + lane; j <= i; j += 32) m = fmax(m, logscore(j));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));

  // pass 2: weights, score sum, weighted values
  T num[kMaxE / 32];
#pragma unroll
  for (int r = 0; r < kMaxE / 32; ++r) num[r] = T(0);
  T wsum = T(0);
  T* wrow = ws + warp * 32;
  for (int j0 = j_lo; j0 <= i; j0 += 32) {
    const int j = j0 + lane;
    T w = (j <= i) ? exp(logscore(j) - m) : T(0);
    wsum += w;
    wrow[lane] = w;
    __syncwarp();
    const int cnt = min(32, i - j0 + 1);
    for (int jj = 0; jj < cnt; ++jj) {
      const T wj = wrow[jj];
      const T* vj = v + (((int64_t)bi * t + j0 + jj) * h + hi) * e;
#pragma unroll
      for (int r = 0; r < kMaxE / 32; ++r) {
        const int c = lane + 32 * r;
        if (c < e) num[r] += wj * vj[c];
      }
    }
    __syncwarp();
  }
  for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);

  const T restore = exp(m);
  T* yi = y + (((int64_t)bi * t + i) * h + hi) * e;
#pragma unroll
  for (int r = 0; r < kMaxE / 32; ++r) {
    const int c = lane + 32 * r;
    if (c < e) yi[c] = normalize ? num[r] / wsum : num[r] * restore;
  }
  if (lane == 0) rowsum[((int64_t)bi * t + i) * h + hi] = wsum * restore;
}

template <typename T>
int launch(const pa_problem* pr, double eps, const void* q, const void* k, const void* v,
           const void* log_g, void* y, void* rowsum, cudaStream_t st) {
  const int t = pr->t;
  size_t smem = (size_t)t * sizeof(double) + (size_t)((t + 1) & ~1) * sizeof(int) +
                (size_t)kRowsPerCta * pr->d * sizeof(T) + (size_t)kRowsPerCta * 32 * sizeof(T);
  if (smem > 200 * 1024) {
    set_error("log-space attention form: t too large for the per-CTA gate prefix (t <= 16384)");
    return PA_ERR_UNSUPPORTED;
  }
  auto kern = k_logspace_attention<T>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return cuda_check("log-space attention smem attribute");
  const T scale = pr->has_scale ? T(pr->scale) : T(1.0 / std::sqrt((double)pr->d));
  dim3 grid((t + kRowsPerCta - 1) / kRowsPerCta, pr->b * pr->h);
  StageTimer tm("fwd_logspace_attention", st);
  kern<<<grid, kThreads, smem, st>>>(t, pr->h, pr->d, pr->e, pr->p, scale, T(eps), pr->normalize,
                                     pr->gated, (const T*)q, (const T*)k, (const T*)v,
                                     (const T*)log_g, (T*)y, (T*)rowsum);
  count_launch();
  return cuda_check("log-space attention launch");
}

}  // namespace
}  // namespace pa

extern "C" int pa_power_logspace_fwd(const pa_problem* pr, double eps, const void* q, const void* k,
                                     const void* v, const void* log_g, void* y, void* rowsum,
                                     pa_stream_t stream) {
  using namespace pa;
  if (!pr || !q || !k || !v || !y || !rowsum || (pr->gated && !log_g)) {
    set_error("null problem or tensor pointer");
    return PA_ERR_SHAPE;
  }
  if (pr->b < 1 || pr->t < 1 || pr->h < 1 || pr->d < 1 || pr->e < 1) {
    set_error("need b, t, h, d, e >= 1");
    return PA_ERR_SHAPE;
  }
  if (pr->p < 2 || pr->p % 2) {
    set_error("log-space scoring needs even p");
    return PA_ERR_INVALID_SPEC;
  }
  if (pr->e > kMaxE || pr->d > 1024) {
    set_error("log-space attention form: e must be <= 128 and d <= 1024");
    return PA_ERR_UNSUPPORTED;
  }
  if (!(eps > 0.0)) {
    set_error("log-space epsilon must be positive");
    return PA_ERR_INVALID_SPEC;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (pr->dtype == PA_F32) return launch<float>(pr, eps, q, k, v, log_g, y, rowsum, st);
  if (pr->dtype == PA_F64) return launch<double>(pr, eps, q, k, v, log_g, y, rowsum, st);
  set_error("log-space attention form takes f32 or f64");
  return PA_ERR_UNSUPPORTED;
}
