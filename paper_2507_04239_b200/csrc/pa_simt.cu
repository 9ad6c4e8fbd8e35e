// FP32 (CUDA-core) kernels for every stage of chunked power attention, forward
// and backward, for any SPOW degree p <= 4 and d, e <= 128.
//
// These are the full-precision path ("fp32 mode", north star: 1e-4 against
// the oracle) and the path for shapes the bf16 tensor-core kernels do not
// specialise.  Each kernel states the reference computation it restates.
//
// Internal layouts (all fp32, stream-major):
//   ell   [ns, t]          inclusive in-chunk cumsum of log g (chunked.py:98-100 in log space)
//   lamlog[ns, n]          log of the chunk total decay lambda_k (chunked.py:279)
//   yat   [ns, t, E1]      intra-chunk output, column e = score sum zeta
//   A     [ns, n, D, E1]   chunk states S_k, then (in place) discumsum A_k; column e = key_sum
#include <algorithm>

#include "pa_common.cuh"
#include "pa_simt.cuh"

namespace pa {

// --------------------------------------------------------------------------
// NDMI table (expansions.py:106-123 order, weights 149-163)
// --------------------------------------------------------------------------
__host__ __device__ inline int64_t binom(int64_t n, int64_t k) {
  if (k < 0 || n < k) return 0;
  if (k > n - k) k = n - k;
  int64_t r = 1;
  for (int64_t i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

__host__ __device__ inline void ndmi_unrank(int64_t r, int p, int d, int* out, float* w) {
  int lo = 0;
  for (int z = 0; z < p; ++z) {
    int rem = p - z - 1;
    for (int a = lo; a < d; ++a) {
      int64_t cnt = binom(d - a + rem - 1, rem);  // tuples of length rem from [a, d)
      if (r < cnt) {
        out[z] = a;
        lo = a;
        break;
      }
      r -= cnt;
    }
  }
  // sqrt(p! / prod hist!) via run lengths
  double fact = 1, den = 1;
  int run = 1;
  for (int z = 1; z <= p; ++z) fact *= z;
  for (int z = 1; z < p; ++z) {
    run = (out[z] == out[z - 1]) ? run + 1 : 1;
    den *= run;
  }
  *w = (float)sqrt(fact / den);
}

__global__ void k_build_table(int p, int d, int D, int* idx, float* wt) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= D) return;
  int o[4] = {0, 0, 0, 0};
  float w;
  ndmi_unrank(f, p, d, o, &w);
  for (int z = 0; z < p; ++z) idx[f * p + z] = o[z];
  wt[f] = w;
}

// TPOW: every ordered tuple, first index slowest, weight 1; TSPOW: one dense
// d_tile^p block per NDMI over tiles, the tile NDMI's weight on the whole block
// (reference expansions.py:171-198).
int64_t host_expansion_dim(int kind, int p, int d, int d_tile) {
  if (kind == 1) {
    int64_t r = 1;
    for (int z = 0; z < p; ++z) r *= d;
    return r;
  }
  if (kind == 2) {
    int64_t r = binom(d / d_tile + p - 1, p);
    for (int z = 0; z < p; ++z) r *= d_tile;
    return r;
  }
  return binom(d + p - 1, p);
}

void host_expansion_table(int kind, int p, int d, int d_tile, int* idx, double* w) {
  if (kind == 0) {
    host_feature_table(p, d, idx, w);
    return;
  }
  if (kind == 1) {
    const int64_t D = host_expansion_dim(1, p, d, 0);
    for (int64_t f = 0; f < D; ++f) {
      int64_t r = f;
      for (int z = p - 1; z >= 0; --z) {
        idx[f * p + z] = (int)(r % d);
        r /= d;
      }
      w[f] = 1.0;
    }
    return;
  }
  const int nt = d / d_tile;
  const int64_t T = binom(nt + p - 1, p), B = host_expansion_dim(1, p, d_tile, 0);
  int* tidx = new int[T * p];
  double* tw = new double[T];
  host_feature_table(p, nt, tidx, tw);
  for (int64_t ti = 0; ti < T; ++ti)
    for (int64_t o = 0; o < B; ++o) {
      const int64_t f = ti * B + o;
      int64_t r = o;
      for (int z = p - 1; z >= 0; --z) {
        idx[f * p + z] = tidx[ti * p + z] * d_tile + (int)(r % d_tile);
        r /= d_tile;
      }
      w[f] = tw[ti];
    }
  delete[] tidx;
  delete[] tw;
}

void host_feature_table(int p, int d, int* idx, double* w) {
  int64_t D = binom(d + p - 1, p);
  for (int64_t f = 0; f < D; ++f) {
    int o[4] = {0, 0, 0, 0};
    float wf;
    ndmi_unrank(f, p, d, o, &wf);
    double fact = 1, den = 1;
    int run = 1;
    for (int z = 1; z <= p; ++z) fact *= z;
    for (int z = 1; z < p; ++z) {
      run = (o[z] == o[z - 1]) ? run + 1 : 1;
      den *= run;
    }
    for (int z = 0; z < p; ++z) idx[f * p + z] = o[z];
    w[f] = sqrt(fact / den);
  }
}

// phi_f(x) with x in shared memory (row pointer), weight included.
__device__ __forceinline__ float phi_at(const float* xrow, const int* id, float w, int p) {
  float r = w * xrow[id[0]];
  for (int z = 1; z < p; ++z) r *= xrow[id[z]];
  return r;
}

// --------------------------------------------------------------------------
// gate prep: ell = inclusive in-chunk cumsum of log g; lamlog = ell at chunk end
// --------------------------------------------------------------------------
__global__ void k_gate_prep(Geo g, const float* __restrict__ log_g, float* ell, float* lamlog) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.ns * g.n) return;
  int s = idx / g.n, k = idx - s * g.n;
  int s0 = k * g.c, s1 = min(s0 + g.c, g.t);
  float acc = 0.f;
  for (int m = s0; m < s1; ++m) {
    float lg = g.gated ? fmaxf(log_g[rowid(g, s, m)], -80.f) : 0.f;
    acc += lg;
    ell[(size_t)s * g.t + m] = acc;
  }
  lamlog[idx] = acc;
}

// --------------------------------------------------------------------------
// intra-chunk forward (attention.py:273-309 / 253-270, normalize=False):
// yat[i] = sum_{j<=i, same chunk} exp(ell_i - ell_j) (sigma q_i.k_j)^p [v_j, 1]
// --------------------------------------------------------------------------
template <typename T, int DM>
__global__ void __launch_bounds__(64) k_intra_fwd(Geo g, const T* __restrict__ q,
                                                  const T* __restrict__ k, const T* __restrict__ v,
                                                  const float* __restrict__ ell, float* yat) {
  extern __shared__ float sm_dyn[];
  float* sm_ptr = sm_dyn;
  float (*Ks)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (64) * (DM + 1);
  float (*Vs)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (64) * (DM + 1);
  __shared__ float Ls[64];
  const int tpc = (g.c + 63) / 64;
  const int kch = blockIdx.x / tpc, tile = blockIdx.x - kch * tpc, s = blockIdx.y;
  const int s0 = kch * g.c, s1 = min(s0 + g.c, g.t);
  const int q0 = s0 + tile * 64;
  if (q0 >= s1) return;
  const int i = q0 + threadIdx.x;
  const bool act = i < s1;
  float qr[DM], o[DM + 1];
#pragma unroll
  for (int a = 0; a < DM; ++a) qr[a] = (act && a < g.d) ? g.scale * to_f(q[rowid(g, s, i) * g.d + a]) : 0.f;
#pragma unroll
  for (int u = 0; u <= DM; ++u) o[u] = 0.f;
  const float li = act ? ell[(size_t)s * g.t + i] : 0.f;
  const int jend = min(q0 + 64, s1);
  for (int j0 = s0; j0 < jend; j0 += 64) {
    __syncthreads();
    {
      int j = j0 + threadIdx.x;
      bool ok = j < jend;
      for (int a = 0; a < DM; ++a) Ks[threadIdx.x][a] = (ok && a < g.d) ? to_f(k[rowid(g, s, j) * g.d + a]) : 0.f;
      for (int u = 0; u < DM; ++u) Vs[threadIdx.x][u] = (ok && u < g.e) ? to_f(v[rowid(g, s, j) * g.e + u]) : 0.f;
      Ls[threadIdx.x] = ok ? ell[(size_t)s * g.t + j] : 0.f;
    }
    __syncthreads();
    const int jn = min(64, jend - j0);
    for (int jj = 0; jj < jn; ++jj) {
      if (act && j0 + jj <= i) {
        float sd = 0.f;
#pragma unroll
        for (int a = 0; a < DM; ++a) sd += qr[a] * Ks[jj][a];
        const float P = expf(li - Ls[jj]) * ipow(sd, g.p);
#pragma unroll
        for (int u = 0; u < DM; ++u) o[u] += P * Vs[jj][u];
        o[DM] += P;
      }
    }
  }
  if (!act) return;
  float* out = yat + ((size_t)s * g.t + i) * g.E1;
#pragma unroll
  for (int u = 0; u < DM; ++u)
    if (u < g.e) out[u] = o[u];
  out[g.e] = o[DM];
}

// --------------------------------------------------------------------------
// state accumulation (update_state kernels.py:55-83 / _core.pyx:18-43, and
// the dA half of the query-state VJP gradients.py:429-430):
//   out[s, kin-koff, f, u] = sum_{j in chunk kin} wt_j phi_f(xs * x_j) vec_j[u]
// wt mode 0: 1; 1: exp(lamlog_k - ell_j) (suffix decay W_j); 2: exp(ell_j) (prefix gp_j)
// vec: u < ev from vec rows (type TV, leading dim ldv); u == ev -> 1 if ones
// --------------------------------------------------------------------------
template <typename TX, typename TV, int DM>
__global__ void __launch_bounds__(256) k_state_accum(Geo g, const TX* __restrict__ x, float xs,
                                                     int wmode, const float* __restrict__ ell,
                                                     const float* __restrict__ lamlog,
                                                     const TV* __restrict__ vec, int vec_bth, int ldv,
                                                     int ev, int ones, const int* __restrict__ idx,
                                                     const float* __restrict__ wt, int kfirst,
                                                     int koff, float* out) {
  constexpr int UM = (DM + 1 + 7) / 8;
  __shared__ float Xs[32][DM + 1];
  __shared__ float Us[32][DM + 2];
  const int fl = threadIdx.x & 31, ug = threadIdx.x >> 5;
  const int f = blockIdx.x * 32 + fl;
  const int kin = kfirst + blockIdx.y, s = blockIdx.z;
  const int s0 = kin * g.c, s1 = min(s0 + g.c, g.t);
  const int ncol = ev + (ones ? 1 : 0);
  int id[4] = {0, 0, 0, 0};
  float w = 0.f;
  if (f < g.D) {
    for (int z = 0; z < g.p; ++z) id[z] = idx[f * g.p + z];
    w = wt[f];
  }
  const float lend = (wmode == 1) ? lamlog[s * g.n + kin] : 0.f;
  float acc[UM];
#pragma unroll
  for (int i = 0; i < UM; ++i) acc[i] = 0.f;
  Geo gv = g;
  gv.bth = vec_bth;
  for (int j0 = s0; j0 < s1; j0 += 32) {
    __syncthreads();
    for (int el = threadIdx.x; el < 32 * (DM + 1); el += 256) {
      int r = el / (DM + 1), a = el - r * (DM + 1);
      int j = j0 + r;
      bool ok = j < s1;
      float wj = 1.f;
      if (ok && wmode) {
        float lj = ell[(size_t)s * g.t + j];
        wj = (wmode == 1) ? expf(lend - lj) : expf(lj);
      }
      Xs[r][a] = (ok && a < g.d) ? xs * to_f(x[rowid(g, s, j) * g.d + a]) : 0.f;
      float uv = 0.f;
      if (ok && a < ev) uv = to_f(vec[rowid(gv, s, j) * ldv + a]);
      else if (ok && a == ev && ones) uv = 1.f;
      Us[r][a] = uv * wj;
    }
    __syncthreads();
    const int jn = min(32, s1 - j0);
    if (f < g.D) {
      for (int jj = 0; jj < jn; ++jj) {
        const float ph = phi_at(Xs[jj], id, w, g.p);
#pragma unroll
        for (int i = 0; i < UM; ++i) {
          int u = ug + 8 * i;
          if (u < ncol) acc[i] += ph * Us[jj][u];
        }
      }
    }
  }
  if (f >= g.D) return;
  float* o = out + (((size_t)s * g.n + (kin - koff)) * g.D + f) * g.E1;
#pragma unroll
  for (int i = 0; i < UM; ++i) {
    int u = ug + 8 * i;
    if (u < ncol) o[u] = acc[i];
  }
}

// Same contraction, one thread per feature (DM <= 64): phi_f is generated once
// per token and feeds all ncol columns from broadcast LDS.128 reads of the
// staged value row, instead of eight threads each regenerating phi_f for
// every eighth column (3x fewer instructions per feature-token at p = 4).
// features per CTA: the staged token rows are shared by this many features
constexpr int kSaThreads = 256;
template <typename TX, typename TV, int DM>
__global__ void __launch_bounds__(kSaThreads) k_state_accum_f(Geo g, const TX* __restrict__ x, float xs,
                                                       int wmode, const float* __restrict__ ell,
                                                       const float* __restrict__ lamlog,
                                                       const TV* __restrict__ vec, int vec_bth, int ldv,
                                                       int ev, int ones, const int* __restrict__ idx,
                                                       const float* __restrict__ wt, int kfirst,
                                                       int koff, float* out) {
  constexpr int US = (DM + 1 + 3) / 4 * 4;  // value row stride, 16-byte aligned
  __shared__ float Xs[32][DM + 1];
  __shared__ __align__(16) float Us[32][US];
  const int f = blockIdx.x * kSaThreads + threadIdx.x;
  const int kin = kfirst + blockIdx.y, s = blockIdx.z;
  const int s0 = kin * g.c, s1 = min(s0 + g.c, g.t);
  const int ncol = ev + (ones ? 1 : 0);
  int id[4] = {0, 0, 0, 0};
  float w = 0.f;
  if (f < g.D) {
    for (int z = 0; z < g.p; ++z) id[z] = idx[f * g.p + z];
    w = wt[f];
  }
  const float lend = (wmode == 1) ? lamlog[s * g.n + kin] : 0.f;
  float acc[US];
#pragma unroll
  for (int u = 0; u < US; ++u) acc[u] = 0.f;
  Geo gv = g;
  gv.bth = vec_bth;
  for (int j0 = s0; j0 < s1; j0 += 32) {
    __syncthreads();
    for (int el = threadIdx.x; el < 32 * US; el += kSaThreads) {
      int r = el / US, a = el - r * US;
      int j = j0 + r;
      bool ok = j < s1;
      float wj = 1.f;
      if (ok && wmode) {
        float lj = ell[(size_t)s * g.t + j];
        wj = (wmode == 1) ? expf(lend - lj) : expf(lj);
      }
      if (a <= DM) Xs[r][a] = (ok && a < g.d) ? xs * to_f(x[rowid(g, s, j) * g.d + a]) : 0.f;
      float uv = 0.f;
      if (ok && a < ev) uv = to_f(vec[rowid(gv, s, j) * ldv + a]);
      else if (ok && a == ev && ones) uv = 1.f;
      Us[r][a] = uv * wj;
    }
    __syncthreads();
    const int jn = min(32, s1 - j0);
    for (int jj = 0; jj < jn; ++jj) {
      const float ph = phi_at(Xs[jj], id, w, g.p);
      const float4* ur = reinterpret_cast<const float4*>(Us[jj]);
#pragma unroll
      for (int q4 = 0; q4 < DM / 4; ++q4) {  // columns 0..DM-1, then column DM alone
        const float4 u4 = ur[q4];
        acc[4 * q4 + 0] += ph * u4.x;
        acc[4 * q4 + 1] += ph * u4.y;
        acc[4 * q4 + 2] += ph * u4.z;
        acc[4 * q4 + 3] += ph * u4.w;
      }
      acc[DM] += ph * Us[jj][DM];
    }
  }
  if (f >= g.D) return;
  float* o = out + (((size_t)s * g.n + (kin - koff)) * g.D + f) * g.E1;
#pragma unroll
  for (int u = 0; u < US; ++u)
    if (u < ncol) o[u] = acc[u];
}

// --------------------------------------------------------------------------
// discumsum over chunk states (chunked.py:156-176, call 356-367), in place:
//   A[s,k] = lambda_k * A[s,k-1] + A[s,k]   (separate mul and add)
// --------------------------------------------------------------------------
__global__ void k_discumsum_states(Geo g, const float* __restrict__ lamlog, float* A) {
  const size_t per = (size_t)g.D * g.E1;
  const int s = blockIdx.y;
  for (size_t m = blockIdx.x * (size_t)blockDim.x + threadIdx.x; m < per; m += (size_t)gridDim.x * blockDim.x) {
    float* p = A + (size_t)s * g.n * per + m;
    float prev = p[0];
    for (int k = 1; k < g.n; ++k) {
      const float lam = g.gated ? expf(lamlog[s * g.n + k]) : 1.f;
      prev = __fadd_rn(__fmul_rn(lam, prev), p[(size_t)k * per]);
      p[(size_t)k * per] = prev;
    }
  }
}

// The same scan with 4 consecutive entries per thread and SC_PF chunks of loads
// in flight (the one-load-per-iteration loop above is latency-bound).  Needs
// D * E1 % 4 == 0.
constexpr int SC_PF = 4;
__global__ void __launch_bounds__(256) k_discumsum_states4(Geo g, const float* __restrict__ lamlog, float* A) {
  const size_t per4 = (size_t)g.D * g.E1 / 4;
  const int s = blockIdx.y;
  const size_t m4 = blockIdx.x * (size_t)256 + threadIdx.x;
  if (m4 >= per4) return;
  float4* p = (float4*)(A + (size_t)s * g.n * per4 * 4) + m4;
  float4 prev = p[0];
  for (int k0 = 1; k0 < g.n; k0 += SC_PF) {
    float4 x[SC_PF];
#pragma unroll
    for (int i = 0; i < SC_PF; ++i)
      x[i] = k0 + i < g.n ? p[(size_t)(k0 + i) * per4] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < SC_PF; ++i) {
      const int k = k0 + i;
      if (k >= g.n) break;
      const float lam = g.gated ? expf(lamlog[s * g.n + k]) : 1.f;
      prev.x = __fadd_rn(__fmul_rn(lam, prev.x), x[i].x);
      prev.y = __fadd_rn(__fmul_rn(lam, prev.y), x[i].y);
      prev.z = __fadd_rn(__fmul_rn(lam, prev.z), x[i].z);
      prev.w = __fadd_rn(__fmul_rn(lam, prev.w), x[i].w);
      p[(size_t)k * per4] = prev;
    }
  }
}

// --------------------------------------------------------------------------
// query-state + combine + normalize (kernels.py:86-110, chunked.py:372-395):
//   y_i = yat_i + gp_i phi(sigma q_i)^T A_{k-1};  optional y /= rowsum
// --------------------------------------------------------------------------
// tokens per CTA of the query-combine kernel (shares each staged state block)
template <int DM> __host__ __device__ constexpr int qc_tokens() { return DM <= 64 ? 128 : 64; }

template <typename T, int DM>
__global__ void __launch_bounds__(qc_tokens<DM>()) k_query_combine(Geo g, const T* __restrict__ q,
                                                      const float* __restrict__ A,
                                                      const int* __restrict__ idx,
                                                      const float* __restrict__ wt,
                                                      const float* __restrict__ ell,
                                                      const float* __restrict__ yat, T* y,
                                                      float* rowsum, int* zflag, float* y32) {
  extern __shared__ float sm_dyn[];
  float* sm_ptr = sm_dyn;
  constexpr int AS = (DM + 1 + 3) / 4 * 4;  // state_row_stride<DM>()
  float (*As)[AS] = reinterpret_cast<float (*)[AS]>(sm_ptr);  // first: 16-byte aligned rows
  sm_ptr += (32) * AS;
  constexpr int TOK = qc_tokens<DM>();
  float (*Qs)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (TOK) * (DM + 1);
  __shared__ int Is[32][4];
  __shared__ float Ws[32];
  const int tpc = (g.c + TOK - 1) / TOK;
  const int kch = blockIdx.x / tpc, tile = blockIdx.x - kch * tpc, s = blockIdx.y;
  const int s0 = kch * g.c, s1 = min(s0 + g.c, g.t);
  const int q0 = s0 + tile * TOK;
  if (q0 >= s1) return;
  const int i = q0 + threadIdx.x;
  const bool act = i < s1;
  for (int a = 0; a < DM; ++a) Qs[threadIdx.x][a] = (act && a < g.d) ? g.scale * to_f(q[rowid(g, s, i) * g.d + a]) : 0.f;
  float acc[AS], accs = 0.f;  // state columns (score column e included) | score sum
#pragma unroll
  for (int u = 0; u < AS; ++u) acc[u] = 0.f;
  if (kch >= 1) {
    const float* Ak = A + ((size_t)s * g.n + (kch - 1)) * g.D * g.E1;
    for (int f0 = 0; f0 < g.D; f0 += 32) {
      __syncthreads();
      for (int el = threadIdx.x; el < 32 * AS; el += TOK) {
        int r = el / AS, u = el - r * AS;
        As[r][u] = (f0 + r < g.D && u < g.E1) ? Ak[(size_t)(f0 + r) * g.E1 + u] : 0.f;
      }
      if (threadIdx.x < 32) {
        int f = f0 + threadIdx.x;
        for (int z = 0; z < 4; ++z) Is[threadIdx.x][z] = (f < g.D && z < g.p) ? idx[f * g.p + z] : 0;
        Ws[threadIdx.x] = f < g.D ? wt[f] : 0.f;
      }
      __syncthreads();
      const int fn = min(32, g.D - f0);
      for (int fl = 0; fl < fn; ++fl) {
        const float ph = phi_at(Qs[threadIdx.x], Is[fl], Ws[fl], g.p);
        const float4* ar = reinterpret_cast<const float4*>(As[fl]);
#pragma unroll
        for (int q4 = 0; q4 < DM / 4; ++q4) {  // y columns are < e <= DM
          const float4 a4 = ar[q4];
          acc[4 * q4] += ph * a4.x;
          acc[4 * q4 + 1] += ph * a4.y;
          acc[4 * q4 + 2] += ph * a4.z;
          acc[4 * q4 + 3] += ph * a4.w;
        }
        accs += ph * As[fl][g.e];
      }
    }
  }
  if (!act) return;
  const float gp = g.gated ? expf(ell[(size_t)s * g.t + i]) : 1.f;
  const float* ya = yat + ((size_t)s * g.t + i) * g.E1;
  const float R = ya[g.e] + gp * accs;
  const size_t r = rowid(g, s, i);
  if (rowsum) rowsum[r] = R;
  float inv = 1.f;
  if (g.normalize) {
    if (!(R > 0.f)) atomicAdd(zflag, 1);
    inv = 1.f / R;
  }
#pragma unroll
  for (int u = 0; u < DM; ++u)
    if (u < g.e) {
      const float yv = (ya[u] + gp * acc[u]) * inv;
      y[r * g.e + u] = from_f<T>(yv);
      if (g.normalize) y32[((size_t)s * g.t + i) * g.e + u] = yv;
    }
}

// --------------------------------------------------------------------------
// backward prep: dz = [dnum, dden] (gradients.py:381-386)
// --------------------------------------------------------------------------
template <typename T>
__global__ void k_bwd_prep(Geo g, const T* __restrict__ dy, const float* __restrict__ y32,
                           const float* __restrict__ rowsum, float* dz) {
  const size_t n = (size_t)g.ns * g.t;
  for (size_t it = blockIdx.x * (size_t)blockDim.x + threadIdx.x; it < n; it += (size_t)gridDim.x * blockDim.x) {
    const int s = (int)(it / g.t), m = (int)(it - (size_t)s * g.t);
    const size_t r = rowid(g, s, m);
    float* o = dz + it * g.E1;
    if (g.normalize) {
      const float R = rowsum[r];
      float dot = 0.f;
      for (int u = 0; u < g.e; ++u) {
        const float dyu = to_f(dy[r * g.e + u]);
        dot += dyu * y32[it * g.e + u];
        o[u] = dyu / R;
      }
      o[g.e] = -dot / R;
    } else {
      for (int u = 0; u < g.e; ++u) o[u] = to_f(dy[r * g.e + u]);
      o[g.e] = 0.f;
    }
  }
}

// tokens per CTA of the token-side state VJPs: each staged block of 32 state rows is
// shared by this many tokens (64 at DM = 128, where shared memory limits it)
template <int DM> __host__ __device__ constexpr int ub_tokens() { return DM <= 64 ? 128 : 64; }

// staged state rows [D-block of 32][AS]: e + 1 columns padded with zeros to a
// multiple of four floats, so the token-side kernels read them as LDS.128
template <int DM> __host__ __device__ constexpr int state_row_stride() { return (DM + 1 + 3) / 4 * 4; }

// accumulate d phi_f into dx (expand_vjp, gradients.py:46-76) -- shared row
__device__ __forceinline__ void phi_vjp_add(const float* xrow, float* dxrow, const int* id, float gw,
                                            int p) {
  if (p == 1) {
    dxrow[id[0]] += gw;
    return;
  }
  for (int z = 0; z < p; ++z) {
    float pr = gw;
    for (int z2 = 0; z2 < p; ++z2)
      if (z2 != z) pr *= xrow[id[z2]];
    dxrow[id[z]] += pr;
  }
}

// phi_f and its expand-VJP from one read of the p coordinates: the partial
// derivatives are products of the other three factors (padded with ones for
// z >= p), formed from pairwise products instead of p reloads per factor.
struct PhiParts {
  float ph, d[4];
};
__device__ __forceinline__ PhiParts phi_parts(const float* xrow, const int* id, float w, int p) {
  float x[4];
#pragma unroll
  for (int z = 0; z < 4; ++z) x[z] = z < p ? xrow[id[z]] : 1.f;
  const float p01 = x[0] * x[1], p23 = x[2] * x[3];
  PhiParts r;
  r.ph = w * p01 * p23;
  r.d[0] = x[1] * p23;
  r.d[1] = x[0] * p23;
  r.d[2] = p01 * x[3];
  r.d[3] = p01 * x[2];
  return r;
}
__device__ __forceinline__ void phi_parts_vjp_add(float* dxrow, const int* id, const PhiParts& pp,
                                                  float gw, int p) {
#pragma unroll
  for (int z = 0; z < 4; ++z)
    if (z < p) dxrow[id[z]] += gw * pp.d[z];
}

// --------------------------------------------------------------------------
// query-state backward, token side (gradients.py:406-431):
//   t_f = A_{k-1}[f,:] . dz_i ; dq_i += sigma * expand_vjp(sigma q_i, gp_i t)
//   dell_i += gp_i * sum_f phi_f(sigma q_i) t_f      (gate prefix, 260-264)
// --------------------------------------------------------------------------
template <typename T, int DM>
__global__ void __launch_bounds__(ub_tokens<DM>()) k_query_bwd(Geo g, const T* __restrict__ q,
                                                  const float* __restrict__ A,
                                                  const int* __restrict__ idx,
                                                  const float* __restrict__ wt,
                                                  const float* __restrict__ ell,
                                                  const float* __restrict__ dz, float* dq32,
                                                  float* dell) {
  extern __shared__ float sm_dyn[];
  float* sm_ptr = sm_dyn;
  constexpr int AS = state_row_stride<DM>();
  float (*As)[AS] = reinterpret_cast<float (*)[AS]>(sm_ptr);  // first: 16-byte aligned rows
  sm_ptr += (32) * AS;
  constexpr int TOK = ub_tokens<DM>();
  float (*Qs)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (TOK) * (DM + 1);
  float (*Dq)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (TOK) * (DM + 1);
  __shared__ int Is[32][4];
  __shared__ float Ws[32];
  const int tpc = (g.c + TOK - 1) / TOK;
  const int kch = 1 + blockIdx.x / tpc, tile = blockIdx.x % tpc, s = blockIdx.y;
  const int s0 = kch * g.c, s1 = min(s0 + g.c, g.t);
  const int q0 = s0 + tile * TOK;
  if (q0 >= s1) return;
  const int i = q0 + threadIdx.x;
  const bool act = i < s1;
  for (int a = 0; a <= DM; ++a) {
    Qs[threadIdx.x][a] = (act && a < g.d) ? g.scale * to_f(q[rowid(g, s, i) * g.d + a]) : 0.f;
    Dq[threadIdx.x][a] = 0.f;
  }
  // dz row in state-column order: [dnum (e) | dden | 0 ...] (AS columns)
  float dzr[AS];
#pragma unroll
  for (int u = 0; u < AS; ++u) dzr[u] = 0.f;
  if (act) {
    const float* dzi = dz + ((size_t)s * g.t + i) * g.E1;
#pragma unroll
    for (int u = 0; u < AS; ++u)
      if (u <= g.e) dzr[u] = dzi[u];
  }
  const float gp = (act && g.gated) ? expf(ell[(size_t)s * g.t + i]) : 1.f;
  float dl = 0.f;
  const float* Ak = A + ((size_t)s * g.n + (kch - 1)) * g.D * g.E1;
  for (int f0 = 0; f0 < g.D; f0 += 32) {
    __syncthreads();
    for (int el = threadIdx.x; el < 32 * AS; el += TOK) {
      int r = el / AS, u = el - r * AS;
      As[r][u] = (f0 + r < g.D && u < g.E1) ? Ak[(size_t)(f0 + r) * g.E1 + u] : 0.f;
    }
    if (threadIdx.x < 32) {
      int f = f0 + threadIdx.x;
      for (int z = 0; z < 4; ++z) Is[threadIdx.x][z] = (f < g.D && z < g.p) ? idx[f * g.p + z] : 0;
      Ws[threadIdx.x] = f < g.D ? wt[f] : 0.f;
    }
    __syncthreads();
    const int fn = min(32, g.D - f0);
    for (int fl = 0; fl < fn; ++fl) {
      const float4* ar = reinterpret_cast<const float4*>(As[fl]);
      float tf = 0.f, tf2 = 0.f;
#pragma unroll
      for (int q4 = 0; q4 < DM / 4; ++q4) {
        const float4 a4 = ar[q4];
        tf += a4.x * dzr[4 * q4] + a4.z * dzr[4 * q4 + 2];
        tf2 += a4.y * dzr[4 * q4 + 1] + a4.w * dzr[4 * q4 + 3];
      }
      tf += tf2 + As[fl][DM] * dzr[DM];  // column DM: the score column when e = DM, else 0
      const PhiParts pp = phi_parts(Qs[threadIdx.x], Is[fl], Ws[fl], g.p);
      dl += pp.ph * tf;
      phi_parts_vjp_add(Dq[threadIdx.x], Is[fl], pp, Ws[fl] * gp * tf, g.p);
    }
  }
  if (!act) return;
  float* o = dq32 + ((size_t)s * g.t + i) * g.d;
  for (int a = 0; a < g.d; ++a) o[a] += g.scale * Dq[threadIdx.x][a];
  dell[(size_t)s * g.t + i] += gp * dl;
}

// --------------------------------------------------------------------------
// discumsum backward in place (gradients.py:267-288) + d lambda reduction:
//   dS_k = dA_k + lambda_{k+1} dS_{k+1};  dlam_{k+1} += <A_k, dS_{k+1}>
// --------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_discumsum_bwd(Geo g, const float* __restrict__ lamlog,
                                                       const float* __restrict__ A, float* dA,
                                                       float* dlam) {
  __shared__ float red[32];
  const size_t per = (size_t)g.D * g.E1;
  const int s = blockIdx.y;
  const size_t m = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const bool ok = m < per;
  const float* Ap = A + (size_t)s * g.n * per + m;
  float* dp = dA + (size_t)s * g.n * per + m;
  float acc = ok ? dp[(size_t)(g.n - 1) * per] : 0.f;
  for (int k = g.n - 2; k >= 0; --k) {
    const float part = ok ? Ap[(size_t)k * per] * acc : 0.f;
    const float tot = block_sum(part, red);
    if (threadIdx.x == 0) atomicAdd(dlam + s * g.n + k + 1, tot);
    const float lam = g.gated ? expf(lamlog[s * g.n + k + 1]) : 1.f;
    if (ok) {
      acc = dp[(size_t)k * per] + lam * acc;
      dp[(size_t)k * per] = acc;
    }
  }
}

// --------------------------------------------------------------------------
// update-state backward, token side (gradients.py:191-213, 245-257):
//   t_f = dS_k[f,:] . [v_j,1];  dk_j += expand_vjp(k_j, W_j t);  dv_j += W_j phi(k_j)^T dS_k
//   dW_j = phi(k_j).t  ->  dell_j -= W_j dW_j,  dell_end(k) += W_j dW_j
// --------------------------------------------------------------------------
template <typename T, int DM>
__global__ void __launch_bounds__(ub_tokens<DM>()) k_update_bwd(Geo g, const T* __restrict__ k,
                                                   const T* __restrict__ v,
                                                   const float* __restrict__ dS,
                                                   const int* __restrict__ idx,
                                                   const float* __restrict__ wt,
                                                   const float* __restrict__ ell,
                                                   const float* __restrict__ lamlog, float* dk32,
                                                   float* dv32, float* dell, float* dellend) {
  extern __shared__ float sm_dyn[];
  float* sm_ptr = sm_dyn;
  constexpr int AS = state_row_stride<DM>();
  float (*Ss)[AS] = reinterpret_cast<float (*)[AS]>(sm_ptr);  // first: 16-byte aligned rows
  sm_ptr += (32) * AS;
  constexpr int TOK = ub_tokens<DM>();
  float (*Ks)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (TOK) * (DM + 1);
  float (*Dk)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (TOK) * (DM + 1);
  __shared__ int Is[32][4];
  __shared__ float Ws[32];
  __shared__ float red[32];
  const int tpc = (g.c + TOK - 1) / TOK;
  const int kch = blockIdx.x / tpc, tile = blockIdx.x % tpc, s = blockIdx.y;
  const int s0 = kch * g.c, s1 = min(s0 + g.c, g.t);
  const int q0 = s0 + tile * TOK;
  if (q0 >= s1) return;
  const int j = q0 + threadIdx.x;
  const bool act = j < s1;
  for (int a = 0; a <= DM; ++a) {
    Ks[threadIdx.x][a] = (act && a < g.d) ? to_f(k[rowid(g, s, j) * g.d + a]) : 0.f;
    Dk[threadIdx.x][a] = 0.f;
  }
  // [v_j | 1 | 0 ...] in state-column order (AS columns)
  float vr[AS], dvr[AS];
#pragma unroll
  for (int u = 0; u < AS; ++u) {
    vr[u] = (act && u < g.e) ? to_f(v[rowid(g, s, j) * g.e + u]) : (u == g.e ? 1.f : 0.f);
    dvr[u] = 0.f;
  }
  const float W = (act && g.gated) ? expf(lamlog[s * g.n + kch] - ell[(size_t)s * g.t + j]) : 1.f;
  float dW = 0.f;
  const float* Sk = dS + ((size_t)s * g.n + kch) * g.D * g.E1;
  for (int f0 = 0; f0 < g.D; f0 += 32) {
    __syncthreads();
    for (int el = threadIdx.x; el < 32 * AS; el += TOK) {
      int r = el / AS, u = el - r * AS;
      Ss[r][u] = (f0 + r < g.D && u < g.E1) ? Sk[(size_t)(f0 + r) * g.E1 + u] : 0.f;
    }
    if (threadIdx.x < 32) {
      int f = f0 + threadIdx.x;
      for (int z = 0; z < 4; ++z) Is[threadIdx.x][z] = (f < g.D && z < g.p) ? idx[f * g.p + z] : 0;
      Ws[threadIdx.x] = f < g.D ? wt[f] : 0.f;
    }
    __syncthreads();
    const int fn = min(32, g.D - f0);
    for (int fl = 0; fl < fn; ++fl) {
      // phi_f depends on k only: one pass over the state row feeds both
      // t_f = S_f . [v|1] and dv += W phi_f S_f
      const PhiParts pp = phi_parts(Ks[threadIdx.x], Is[fl], Ws[fl], g.p);
      const float wp = W * pp.ph;
      const float4* sr = reinterpret_cast<const float4*>(Ss[fl]);
      float tf = 0.f, tf2 = 0.f;
#pragma unroll
      for (int q4 = 0; q4 < DM / 4; ++q4) {  // dv columns are < e <= DM
        const float4 s4 = sr[q4];
        tf += s4.x * vr[4 * q4] + s4.z * vr[4 * q4 + 2];
        tf2 += s4.y * vr[4 * q4 + 1] + s4.w * vr[4 * q4 + 3];
        dvr[4 * q4] += wp * s4.x;
        dvr[4 * q4 + 1] += wp * s4.y;
        dvr[4 * q4 + 2] += wp * s4.z;
        dvr[4 * q4 + 3] += wp * s4.w;
      }
      tf += tf2 + Ss[fl][DM] * vr[DM];  // column DM: the score column when e = DM, else 0
      dW += pp.ph * tf;
      phi_parts_vjp_add(Dk[threadIdx.x], Is[fl], pp, Ws[fl] * W * tf, g.p);
    }
  }
  const float contrib = act ? W * dW : 0.f;
  const float tot = block_sum(contrib, red);
  if (threadIdx.x == 0 && g.gated) atomicAdd(dellend + s * g.n + kch, tot);
  if (!act) return;
  float* ok_ = dk32 + ((size_t)s * g.t + j) * g.d;
  for (int a = 0; a < g.d; ++a) ok_[a] += Dk[threadIdx.x][a];
  float* ov = dv32 + ((size_t)s * g.t + j) * g.e;
#pragma unroll
  for (int u = 0; u < DM; ++u)
    if (u < g.e) ov[u] += dvr[u];
  dell[(size_t)s * g.t + j] -= contrib;
}

// --------------------------------------------------------------------------
// intra-chunk backward (gradients.py:98-176): query side
//   dP_ij = dnum_i . v_j + dden_i;  ds = dP E p s^(p-1);  dq_i += sigma sum_j ds k_j
//   dell_i += sum_j dP_ij P_ij   (pairwise-decay rule 79-95 in log space)
// --------------------------------------------------------------------------
template <typename T, int DM>
__global__ void __launch_bounds__(64) k_intra_bwd_q(Geo g, const T* __restrict__ q,
                                                    const T* __restrict__ k,
                                                    const T* __restrict__ v,
                                                    const float* __restrict__ ell,
                                                    const float* __restrict__ dz, float* dq32,
                                                    float* dell) {
  extern __shared__ float sm_dyn[];
  float* sm_ptr = sm_dyn;
  float (*Ks)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (64) * (DM + 1);
  float (*Vs)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (64) * (DM + 1);
  __shared__ float Ls[64];
  float (*Qr)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (64) * (DM + 1);
  float (*Zr)[DM + 2] = reinterpret_cast<float (*)[DM + 2]>(sm_ptr);
  sm_ptr += (64) * (DM + 2);
  const int tpc = (g.c + 63) / 64;
  const int kch = blockIdx.x / tpc, tile = blockIdx.x - kch * tpc, s = blockIdx.y;
  const int s0 = kch * g.c, s1 = min(s0 + g.c, g.t);
  const int q0 = s0 + tile * 64;
  if (q0 >= s1) return;
  const int i = q0 + threadIdx.x;
  const bool act = i < s1;
  for (int a = 0; a < DM; ++a) Qr[threadIdx.x][a] = (act && a < g.d) ? g.scale * to_f(q[rowid(g, s, i) * g.d + a]) : 0.f;
  for (int u = 0; u <= DM; ++u) {
    float val = 0.f;
    if (act && u < g.e) val = dz[((size_t)s * g.t + i) * g.E1 + u];
    if (act && u == DM) val = dz[((size_t)s * g.t + i) * g.E1 + g.e];
    Zr[threadIdx.x][u] = val;
  }
  float dqa[DM];
#pragma unroll
  for (int a = 0; a < DM; ++a) dqa[a] = 0.f;
  float rowD = 0.f;
  const float li = act ? ell[(size_t)s * g.t + i] : 0.f;
  const int jend = min(q0 + 64, s1);
  for (int j0 = s0; j0 < jend; j0 += 64) {
    __syncthreads();
    {
      int j = j0 + threadIdx.x;
      bool ok = j < jend;
      for (int a = 0; a < DM; ++a) Ks[threadIdx.x][a] = (ok && a < g.d) ? to_f(k[rowid(g, s, j) * g.d + a]) : 0.f;
      for (int u = 0; u < DM; ++u) Vs[threadIdx.x][u] = (ok && u < g.e) ? to_f(v[rowid(g, s, j) * g.e + u]) : 0.f;
      Ls[threadIdx.x] = ok ? ell[(size_t)s * g.t + j] : 0.f;
    }
    __syncthreads();
    const int jn = min(64, jend - j0);
    for (int jj = 0; jj < jn; ++jj) {
      if (act && j0 + jj <= i) {
        float sd = 0.f;
        for (int a = 0; a < DM; ++a) sd += Qr[threadIdx.x][a] * Ks[jj][a];
        float dP = Zr[threadIdx.x][DM];
        for (int u = 0; u < DM; ++u) dP += Zr[threadIdx.x][u] * Vs[jj][u];
        const float E = expf(li - Ls[jj]);
        const float sp1 = ipow(sd, g.p - 1);
        rowD += dP * E * sp1 * sd;
        const float ds = dP * E * g.p * sp1;
#pragma unroll
        for (int a = 0; a < DM; ++a) dqa[a] += ds * Ks[jj][a];
      }
    }
  }
  if (!act) return;
  float* o = dq32 + ((size_t)s * g.t + i) * g.d;
  for (int a = 0; a < DM; ++a)
    if (a < g.d) o[a] += g.scale * dqa[a];
  dell[(size_t)s * g.t + i] += rowD;
}

// key side: dv_j += sum_i P_ij dnum_i; dk_j += sum_i ds_ij (sigma q_i); dell_j -= sum_i dP_ij P_ij
template <typename T, int DM>
__global__ void __launch_bounds__(64) k_intra_bwd_kv(Geo g, const T* __restrict__ q,
                                                     const T* __restrict__ k,
                                                     const T* __restrict__ v,
                                                     const float* __restrict__ ell,
                                                     const float* __restrict__ dz, float* dk32,
                                                     float* dv32, float* dell) {
  extern __shared__ float sm_dyn[];
  float* sm_ptr = sm_dyn;
  float (*Qs)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (64) * (DM + 1);
  float (*Zs)[DM + 2] = reinterpret_cast<float (*)[DM + 2]>(sm_ptr);
  sm_ptr += (64) * (DM + 2);
  __shared__ float Ls[64];
  float (*Kr)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (64) * (DM + 1);
  float (*Vr)[DM + 1] = reinterpret_cast<float (*)[DM + 1]>(sm_ptr);
  sm_ptr += (64) * (DM + 1);
  const int tpc = (g.c + 63) / 64;
  const int kch = blockIdx.x / tpc, tile = blockIdx.x - kch * tpc, s = blockIdx.y;
  const int s0 = kch * g.c, s1 = min(s0 + g.c, g.t);
  const int k0 = s0 + tile * 64;
  if (k0 >= s1) return;
  const int j = k0 + threadIdx.x;
  const bool act = j < s1;
  for (int a = 0; a < DM; ++a) {
    Kr[threadIdx.x][a] = (act && a < g.d) ? to_f(k[rowid(g, s, j) * g.d + a]) : 0.f;
    Vr[threadIdx.x][a] = (act && a < g.e) ? to_f(v[rowid(g, s, j) * g.e + a]) : 0.f;
  }
  float dka[DM], dva[DM];
#pragma unroll
  for (int a = 0; a < DM; ++a) dka[a] = dva[a] = 0.f;
  float colD = 0.f;
  const float lj = act ? ell[(size_t)s * g.t + j] : 0.f;
  for (int i0 = k0; i0 < s1; i0 += 64) {
    __syncthreads();
    {
      int i = i0 + threadIdx.x;
      bool ok = i < s1;
      for (int a = 0; a < DM; ++a) Qs[threadIdx.x][a] = (ok && a < g.d) ? g.scale * to_f(q[rowid(g, s, i) * g.d + a]) : 0.f;
      for (int u = 0; u <= DM; ++u) {
        float val = 0.f;
        if (ok && u < g.e) val = dz[((size_t)s * g.t + i) * g.E1 + u];
        if (ok && u == DM) val = dz[((size_t)s * g.t + i) * g.E1 + g.e];
        Zs[threadIdx.x][u] = val;
      }
      Ls[threadIdx.x] = ok ? ell[(size_t)s * g.t + i] : 0.f;
    }
    __syncthreads();
    const int in = min(64, s1 - i0);
    for (int ii = 0; ii < in; ++ii) {
      if (act && i0 + ii >= j) {
        float sd = 0.f;
        for (int a = 0; a < DM; ++a) sd += Qs[ii][a] * Kr[threadIdx.x][a];
        float dP = Zs[ii][DM];
        for (int u = 0; u < DM; ++u) dP += Zs[ii][u] * Vr[threadIdx.x][u];
        const float E = expf(Ls[ii] - lj);
        const float sp1 = ipow(sd, g.p - 1);
        const float P = E * sp1 * sd;
        colD += dP * P;
        const float ds = dP * E * g.p * sp1;
#pragma unroll
        for (int a = 0; a < DM; ++a) {
          dka[a] += ds * Qs[ii][a];
          dva[a] += P * Zs[ii][a];
        }
      }
    }
  }
  if (!act) return;
  float* ok_ = dk32 + ((size_t)s * g.t + j) * g.d;
  float* ov = dv32 + ((size_t)s * g.t + j) * g.e;
  for (int a = 0; a < DM; ++a) {
    if (a < g.d) ok_[a] += dka[a];
    if (a < g.e) ov[a] += dva[a];
  }
  dell[(size_t)s * g.t + j] -= colD;
}

// --------------------------------------------------------------------------
// gate finish: dlog g_u = sum_{m >= u in chunk} dell_m, with the chunk-end
// cotangents (suffix decay + lambda) folded into the last token.
// --------------------------------------------------------------------------
__global__ void k_gate_finish(Geo g, const float* __restrict__ lamlog, const float* __restrict__ dell,
                              const float* __restrict__ dellend, const float* __restrict__ dlam,
                              float* dlogg) {
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= g.ns * g.n) return;
  int s = idx / g.n, kch = idx - s * g.n;
  int s0 = kch * g.c, s1 = min(s0 + g.c, g.t);
  float acc = dellend[idx] + (kch >= 1 ? dlam[idx] * expf(lamlog[idx]) : 0.f);
  for (int m = s1 - 1; m >= s0; --m) {
    acc += dell[(size_t)s * g.t + m];
    dlogg[rowid(g, s, m)] = acc;
  }
}

template <typename T>
__global__ void k_finalize(Geo g, const float* __restrict__ src, int w, T* dst) {
  const size_t n = (size_t)g.ns * g.t * w;
  for (size_t it = blockIdx.x * (size_t)blockDim.x + threadIdx.x; it < n; it += (size_t)gridDim.x * blockDim.x) {
    const size_t tok = it / w;
    const int col = (int)(it - tok * w);
    const int s = (int)(tok / g.t), m = (int)(tok - (size_t)s * g.t);
    dst[rowid(g, s, m) * w + col] = from_f<T>(src[it]);
  }
}

// --------------------------------------------------------------------------
// public per-operator kernels (reference kernels.py / _core.pyx), f32 or f64
// --------------------------------------------------------------------------
template <typename A>
__global__ void k_pub_update(int n, int c, int d, int e, int p, int D, const A* __restrict__ k,
                             const A* __restrict__ v, const A* __restrict__ w,
                             const int* __restrict__ idx, const double* __restrict__ wt, A* state,
                             A* key_sum, int accumulate) {
  // one thread per (stream, feature, column): the reference's _core.update_state
  // loop nest (_core.pyx:18-43) with the caller's monomial table (idx, weights)
  const size_t tot = (size_t)n * D * (e + 1);
  for (size_t it = blockIdx.x * (size_t)blockDim.x + threadIdx.x; it < tot; it += (size_t)gridDim.x * blockDim.x) {
    const int u = (int)(it % (e + 1));
    const size_t sf = it / (e + 1);
    const int f = (int)(sf % D), s = (int)(sf / D);
    int id[4] = {0, 0, 0, 0};
    for (int z = 0; z < p; ++z) id[z] = idx[(size_t)f * p + z];
    const A wf = (A)wt[f];
    A acc = 0;
    for (int j = 0; j < c; ++j) {
      const A* kr = k + ((size_t)s * c + j) * d;
      A ph = wf * kr[id[0]];
      for (int z = 1; z < p; ++z) ph *= kr[id[z]];
      if (w) ph *= w[(size_t)s * c + j];
      acc += (u < e) ? ph * v[((size_t)s * c + j) * e + u] : ph;
    }
    A* o = (u < e) ? state + ((size_t)s * D + f) * e + u : key_sum + (size_t)s * D + f;
    *o = accumulate ? *o + acc : acc;
  }
}

template <typename A>
__global__ void k_pub_query(int n, int c, int d, int e, int p, int D, const A* __restrict__ q,
                            const A* __restrict__ state, const A* __restrict__ key_sum,
                            const int* __restrict__ idx, const double* __restrict__ wt, A* y, A* denom,
                            int accumulate) {
  // one thread per (stream, token, column): _core.query_state (_core.pyx:46-64)
  const size_t tot = (size_t)n * c * (e + 1);
  for (size_t it = blockIdx.x * (size_t)blockDim.x + threadIdx.x; it < tot; it += (size_t)gridDim.x * blockDim.x) {
    const int u = (int)(it % (e + 1));
    const size_t sm = it / (e + 1);
    const int m = (int)(sm % c), s = (int)(sm / c);
    const A* qr = q + ((size_t)s * c + m) * d;
    A acc = 0;
    for (int f = 0; f < D; ++f) {
      A ph = (A)wt[f] * qr[idx[(size_t)f * p]];
      for (int z = 1; z < p; ++z) ph *= qr[idx[(size_t)f * p + z]];
      acc += ph * ((u < e) ? state[((size_t)s * D + f) * e + u] : key_sum[(size_t)s * D + f]);
    }
    A* o = (u < e) ? y + ((size_t)s * c + m) * e + u : denom + (size_t)s * c + m;
    *o = accumulate ? *o + acc : acc;
  }
}

template <typename A>
__global__ void k_pub_discumsum(int n, int64_t L, int64_t M, const A* __restrict__ values,
                                const A* __restrict__ lams, A* out) {
  const size_t tot = (size_t)L * M;
  for (size_t it = blockIdx.x * (size_t)blockDim.x + threadIdx.x; it < tot; it += (size_t)gridDim.x * blockDim.x) {
    const size_t l = it / M;
    A prev = values[it];
    out[it] = prev;
    for (int k = 1; k < n; ++k) {
      const A lam = lams[(size_t)(k - 1) * L + l];
      A prod;
      if constexpr (sizeof(A) == 8) {
        prod = __dmul_rn(lam, prev);
        prev = __dadd_rn(prod, values[(size_t)k * tot + it]);
      } else {
        prod = __fmul_rn(lam, prev);
        prev = __fadd_rn(prod, values[(size_t)k * tot + it]);
      }
      out[(size_t)k * tot + it] = prev;
    }
  }
}

// ==========================================================================
// host launchers
// ==========================================================================

// --------------------------------------------------------------------------
// d = e = 32 (configs[2]) variants of the three intra-chunk kernels above with
// the same math and tiling: TPR threads per row (each owns 32 / TPR of the dims,
// each dot product combined with log2(TPR) shuffles), the row's
// operands in registers and the shared key / query rows read as broadcast
// float4s (the generic kernels re-read every operand as scalars from shared
// memory).  64 x TPR threads = 64 rows per CTA.
// --------------------------------------------------------------------------
template <int N, typename T>
__device__ __forceinline__ void load_part(const T* src, float sc, float* dst) {
#pragma unroll
  for (int a = 0; a < N; ++a) dst[a] = sc * to_f(src[a]);
}
// 64 rows x 32 values into float4 smem rows, TPR threads per row
template <int TPR, typename T>
__device__ __forceinline__ void stage_rows_p(float4 (*dst)[8], const T* base, const Geo& g, int s, int j0, int jend,
                                             float sc) {
  constexpr int DP = 32 / TPR;
  const int r = threadIdx.x / TPR, hf = threadIdx.x % TPR, j = j0 + r;
  const bool ok = j < jend;
  float v[DP];
  if (ok) load_part<DP>(base + rowid(g, s, j) * 32 + DP * hf, sc, v);
#pragma unroll
  for (int c = 0; c < DP / 4; ++c)
    dst[r][(DP / 4) * hf + c] = ok ? make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
}
template <int DP>
__device__ __forceinline__ float dot_part(const float* x, const float4* y) {
  float p[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int c = 0; c < DP / 4; ++c) {
    const float4 v = y[c];
    p[0] = fmaf(x[4 * c], v.x, p[0]);
    p[1] = fmaf(x[4 * c + 1], v.y, p[1]);
    p[2] = fmaf(x[4 * c + 2], v.z, p[2]);
    p[3] = fmaf(x[4 * c + 3], v.w, p[3]);
  }
  return (p[0] + p[1]) + (p[2] + p[3]);
}
template <int TPR>
__device__ __forceinline__ float row_sum(float v) {
#pragma unroll
  for (int o = 1; o < TPR; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <int DP>
__device__ __forceinline__ void axpy_part(float a, const float4* y, float* acc) {
#pragma unroll
  for (int c = 0; c < DP / 4; ++c) {
    const float4 v = y[c];
    acc[4 * c] = fmaf(a, v.x, acc[4 * c]);
    acc[4 * c + 1] = fmaf(a, v.y, acc[4 * c + 1]);
    acc[4 * c + 2] = fmaf(a, v.z, acc[4 * c + 2]);
    acc[4 * c + 3] = fmaf(a, v.w, acc[4 * c + 3]);
  }
}

template <typename T, int TPR>
__global__ void __launch_bounds__(64 * TPR) k_intra_fwd_h(Geo g, const T* __restrict__ q, const T* __restrict__ k,
                                                          const T* __restrict__ v, const float* __restrict__ ell,
                                                          float* yat) {
  constexpr int DP = 32 / TPR;
  __shared__ float4 Ks[64][8], Vs[64][8];
  __shared__ float Ls[64];
  const int tpc = (g.c + 63) / 64;
  const int kch = blockIdx.x / tpc, tile = blockIdx.x - kch * tpc, s = blockIdx.y;
  const int s0 = kch * g.c, s1 = min(s0 + g.c, g.t);
  const int q0 = s0 + tile * 64;
  if (q0 >= s1) return;
  const int hf = threadIdx.x % TPR, i = q0 + threadIdx.x / TPR;
  const bool act = i < s1;
  float qr[DP], o[DP], rs = 0.f;
#pragma unroll
  for (int a = 0; a < DP; ++a) qr[a] = o[a] = 0.f;
  if (act) load_part<DP>(q + rowid(g, s, i) * 32 + DP * hf, g.scale, qr);
  const float li = act ? ell[(size_t)s * g.t + i] : 0.f;
  const int jend = min(q0 + 64, s1);
  for (int j0 = s0; j0 < jend; j0 += 64) {
    __syncthreads();
    stage_rows_p<TPR>(Ks, k, g, s, j0, jend, 1.f);
    stage_rows_p<TPR>(Vs, v, g, s, j0, jend, 1.f);
    if (threadIdx.x < 64) Ls[threadIdx.x] = j0 + threadIdx.x < jend ? ell[(size_t)s * g.t + j0 + threadIdx.x] : 0.f;
    __syncthreads();
    const int jn = min(64, jend - j0);
    for (int jj = 0; jj < jn; ++jj) {
      const float sd = row_sum<TPR>(dot_part<DP>(qr, &Ks[jj][(DP / 4) * hf]));
      if (act && j0 + jj <= i) {
        const float P = expf(li - Ls[jj]) * ipow(sd, g.p);
        axpy_part<DP>(P, &Vs[jj][(DP / 4) * hf], o);
        rs += P;
      }
    }
  }
  if (!act) return;
  float* out = yat + ((size_t)s * g.t + i) * 33 + DP * hf;
#pragma unroll
  for (int u = 0; u < DP; ++u) out[u] = o[u];
  if (hf == TPR - 1) out[DP] = rs;
}

template <typename T, int TPR>
__global__ void __launch_bounds__(64 * TPR) k_intra_bwd_q_h(Geo g, const T* __restrict__ q, const T* __restrict__ k,
                                                            const T* __restrict__ v, const float* __restrict__ ell,
                                                            const float* __restrict__ dz, float* dq32, float* dell) {
  constexpr int DP = 32 / TPR;
  __shared__ float4 Ks[64][8], Vs[64][8];
  __shared__ float Ls[64];
  const int tpc = (g.c + 63) / 64;
  const int kch = blockIdx.x / tpc, tile = blockIdx.x - kch * tpc, s = blockIdx.y;
  const int s0 = kch * g.c, s1 = min(s0 + g.c, g.t);
  const int q0 = s0 + tile * 64;
  if (q0 >= s1) return;
  const int hf = threadIdx.x % TPR, i = q0 + threadIdx.x / TPR;
  const bool act = i < s1;
  float qr[DP], zr[DP], dqa[DP], zd = 0.f;
#pragma unroll
  for (int a = 0; a < DP; ++a) qr[a] = zr[a] = dqa[a] = 0.f;
  if (act) {
    load_part<DP>(q + rowid(g, s, i) * 32 + DP * hf, g.scale, qr);
    const float* zp = dz + ((size_t)s * g.t + i) * 33;
#pragma unroll
    for (int u = 0; u < DP; ++u) zr[u] = zp[DP * hf + u];
    if (!hf) zd = zp[32];   // dden, added once per pair
  }
  float rowD = 0.f;
  const float li = act ? ell[(size_t)s * g.t + i] : 0.f;
  const int jend = min(q0 + 64, s1);
  for (int j0 = s0; j0 < jend; j0 += 64) {
    __syncthreads();
    stage_rows_p<TPR>(Ks, k, g, s, j0, jend, 1.f);
    stage_rows_p<TPR>(Vs, v, g, s, j0, jend, 1.f);
    if (threadIdx.x < 64) Ls[threadIdx.x] = j0 + threadIdx.x < jend ? ell[(size_t)s * g.t + j0 + threadIdx.x] : 0.f;
    __syncthreads();
    const int jn = min(64, jend - j0);
    for (int jj = 0; jj < jn; ++jj) {
      const float sd = row_sum<TPR>(dot_part<DP>(qr, &Ks[jj][(DP / 4) * hf]));
      const float dP = row_sum<TPR>(zd + dot_part<DP>(zr, &Vs[jj][(DP / 4) * hf]));
      if (act && j0 + jj <= i) {
        const float E = expf(li - Ls[jj]);
        const float sp1 = ipow(sd, g.p - 1);
        rowD += dP * E * sp1 * sd;
        axpy_part<DP>(dP * E * g.p * sp1, &Ks[jj][(DP / 4) * hf], dqa);
      }
    }
  }
  if (!act) return;
  float* o = dq32 + ((size_t)s * g.t + i) * 32 + DP * hf;
#pragma unroll
  for (int a = 0; a < DP; ++a) o[a] += g.scale * dqa[a];
  if (!hf) dell[(size_t)s * g.t + i] += rowD;
}

template <typename T, int TPR>
__global__ void __launch_bounds__(64 * TPR) k_intra_bwd_kv_h(Geo g, const T* __restrict__ q, const T* __restrict__ k,
                                                             const T* __restrict__ v, const float* __restrict__ ell,
                                                             const float* __restrict__ dz, float* dk32, float* dv32,
                                                             float* dell) {
  constexpr int DP = 32 / TPR;
  __shared__ float4 Qs[64][8], Zs[64][8];
  __shared__ float Zd[64], Ls[64];
  const int tpc = (g.c + 63) / 64;
  const int kch = blockIdx.x / tpc, tile = blockIdx.x - kch * tpc, s = blockIdx.y;
  const int s0 = kch * g.c, s1 = min(s0 + g.c, g.t);
  const int k0 = s0 + tile * 64;
  if (k0 >= s1) return;
  const int hf = threadIdx.x % TPR, j = k0 + threadIdx.x / TPR;
  const bool act = j < s1;
  float kr[DP], vr[DP], dka[DP], dva[DP];
#pragma unroll
  for (int a = 0; a < DP; ++a) kr[a] = vr[a] = dka[a] = dva[a] = 0.f;
  if (act) {
    load_part<DP>(k + rowid(g, s, j) * 32 + DP * hf, 1.f, kr);
    load_part<DP>(v + rowid(g, s, j) * 32 + DP * hf, 1.f, vr);
  }
  float colD = 0.f;
  const float lj = act ? ell[(size_t)s * g.t + j] : 0.f;
  for (int i0 = k0; i0 < s1; i0 += 64) {
    __syncthreads();
    stage_rows_p<TPR>(Qs, q, g, s, i0, s1, g.scale);
    {
      const int r = threadIdx.x / TPR, i = i0 + r;
      const bool ok = i < s1;
      const float* zp = dz + ((size_t)s * g.t + (ok ? i : 0)) * 33 + DP * hf;
#pragma unroll
      for (int c = 0; c < DP / 4; ++c)
        Zs[r][(DP / 4) * hf + c] = ok ? make_float4(zp[4 * c], zp[4 * c + 1], zp[4 * c + 2], zp[4 * c + 3]) : make_float4(0.f, 0.f, 0.f, 0.f);
      if (hf == 0) Zd[r] = ok ? zp[32] : 0.f;
      if (hf == TPR - 1) Ls[r] = ok ? ell[(size_t)s * g.t + i] : 0.f;
    }
    __syncthreads();
    const int in = min(64, s1 - i0);
    for (int ii = 0; ii < in; ++ii) {
      const float sd = row_sum<TPR>(dot_part<DP>(kr, &Qs[ii][(DP / 4) * hf]));
      const float dP = row_sum<TPR>((hf ? 0.f : Zd[ii]) + dot_part<DP>(vr, &Zs[ii][(DP / 4) * hf]));
      if (act && i0 + ii >= j) {
        const float E = expf(Ls[ii] - lj);
        const float sp1 = ipow(sd, g.p - 1);
        const float P = E * sp1 * sd;
        colD += dP * P;
        axpy_part<DP>(dP * E * g.p * sp1, &Qs[ii][(DP / 4) * hf], dka);
        axpy_part<DP>(P, &Zs[ii][(DP / 4) * hf], dva);
      }
    }
  }
  if (!act) return;
  float* ok_ = dk32 + ((size_t)s * g.t + j) * 32 + DP * hf;
  float* ov = dv32 + ((size_t)s * g.t + j) * 32 + DP * hf;
#pragma unroll
  for (int a = 0; a < DP; ++a) {
    ok_[a] += dka[a];
    ov[a] += dva[a];
  }
  if (!hf) dell[(size_t)s * g.t + j] -= colD;
}

static bool getenv_flag(const char* name) {
  const char* e = getenv(name);
  return e && e[0] == '1';
}
constexpr int kIntraTpr = 2;   // threads per row of the d = 32 intra-chunk kernels (4 measured slower)

// dynamic shared memory per block for the kernels above (floats -> bytes)
template <int DM> constexpr size_t smb_intra_fwd() { return 4 * (2 * 64 * (DM + 1)); }
template <int DM> constexpr size_t smb_query_combine() { return 4 * (qc_tokens<DM>() * (DM + 1) + 32 * state_row_stride<DM>()); }
template <int DM> constexpr size_t smb_query_bwd() { return 4 * (2 * ub_tokens<DM>() * (DM + 1) + 32 * state_row_stride<DM>()); }
template <int DM> constexpr size_t smb_update_bwd() { return 4 * (2 * ub_tokens<DM>() * (DM + 1) + 32 * state_row_stride<DM>()); }
template <int DM> constexpr size_t smb_intra_bwd() { return 4 * (3 * 64 * (DM + 1) + 64 * (DM + 2)); }

template <typename K>
static size_t dyn_smem(K kern, size_t bytes) {
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  return bytes;
}

static inline unsigned nblk(size_t n, int bs) { return (unsigned)std::min<size_t>((n + bs - 1) / bs, 148 * 32); }

int simt_build_table(int p, int d, int D, int* idx, float* wt, cudaStream_t st) {
  k_build_table<<<(D + 127) / 128, 128, 0, st>>>(p, d, D, idx, wt);
  count_launch();
  return cuda_check("build_table");
}

template <typename T, int DM>
static int simt_forward_t(const Geo& g, const T* q, const T* k, const T* v, const float* log_g, T* y,
                          float* rowsum, const SimtWs& w, cudaStream_t st) {
  const int tpc = (g.c + 63) / 64;
  k_gate_prep<<<(g.ns * g.n + 127) / 128, 128, 0, st>>>(g, log_g, w.ell, w.lamlog);
  int intra_rc = 1;
  if (tc4_supported(g, g.dtype)) {
    intra_rc = tc4_intra_fwd(g, q, k, v, w.ell, w.yat, w.tc4, st);
    if (intra_rc > 1) return intra_rc;
  }
  if (intra_rc == 0) {
  } else if (DM == 32 && g.d == 32 && g.e == 32)
    k_intra_fwd_h<T, kIntraTpr><<<dim3(g.n * tpc, g.ns), 64 * kIntraTpr, 0, st>>>(g, q, k, v, w.ell, w.yat);
  else
    k_intra_fwd<T, DM><<<dim3(g.n * tpc, g.ns), 64, dyn_smem(k_intra_fwd<T, DM>, smb_intra_fwd<DM>()), st>>>(g, q, k, v, w.ell, w.yat);
  if (tc4_supported(g, g.dtype)) {
    if (int rc = tc4_state(g, false, k, v, nullptr, w.ell, w.lamlog, w.idx, w.wt, w.tc4, w.A, st)) return rc;
  } else if constexpr (DM <= 64)
    k_state_accum_f<T, T, DM><<<dim3((g.D + kSaThreads - 1) / kSaThreads, g.n, g.ns), kSaThreads, 0, st>>>(
        g, k, 1.f, g.gated ? 1 : 0, w.ell, w.lamlog, v, 1, g.e, g.e, 1, w.idx, w.wt, 0, 0, w.A);
  else
    k_state_accum<T, T, DM><<<dim3((g.D + 31) / 32, g.n, g.ns), 256, 0, st>>>(
        g, k, 1.f, g.gated ? 1 : 0, w.ell, w.lamlog, v, 1, g.e, g.e, 1, w.idx, w.wt, 0, 0, w.A);
  const bool scan4 = ((size_t)g.D * g.E1) % 4 == 0;
  const bool tc4 = tc4_supported(g, g.dtype);
  if (tc4) {
    // discumsum + fp16 operands in one pass, then the state query + combine on
    // the tensor cores (phi(q) generated on chip)
    if (int rc = tc4_scan_fwd(g, w.lamlog, w.A, w.wt, w.tc4, st)) return rc;
    if (int rc = tc4_tok(g, 0, q, w.ell, w.lamlog, w.yat, y, rowsum, w.y32, w.zflag, nullptr, w.tc4, st)) return rc;
  } else {
  if (scan4 && g.n > 1)
    k_discumsum_states4<<<dim3((unsigned)(((size_t)g.D * g.E1 / 4 + 255) / 256), g.ns), 256, 0, st>>>(
        g, w.lamlog, w.A);
  else if (g.n > 1)
    k_discumsum_states<<<dim3((unsigned)std::min<size_t>(((size_t)g.D * g.E1 + 255) / 256, 512), g.ns), 256, 0, st>>>(g, w.lamlog, w.A);
  k_query_combine<T, DM><<<dim3(g.n * ((g.c + qc_tokens<DM>() - 1) / qc_tokens<DM>()), g.ns), qc_tokens<DM>(),
                           dyn_smem(k_query_combine<T, DM>, smb_query_combine<DM>()), st>>>(g, q, w.A, w.idx, w.wt, w.ell, w.yat, y, rowsum, w.zflag, w.y32);
  }
  count_launch(g.n > 1 ? 5 : 4);
  return cuda_check("simt forward");
}

template <typename T, int DM>
static int simt_backward_t(const Geo& g, const T* q, const T* k, const T* v, const T* y,
                           const float* rowsum, const T* dy, T* dq, T* dk, T* dv, float* dlogg,
                           const SimtWs& w, const SimtBwdWs& b, cudaStream_t st) {
  const int tpc = (g.c + 63) / 64;
  const size_t per = (size_t)g.D * g.E1;
  cudaMemsetAsync(b.dA, 0, sizeof(float) * g.ns * g.n * per, st);
  cudaMemsetAsync(b.dq32, 0, sizeof(float) * g.ns * g.t * g.d, st);
  cudaMemsetAsync(b.dk32, 0, sizeof(float) * g.ns * g.t * g.d, st);
  cudaMemsetAsync(b.dv32, 0, sizeof(float) * g.ns * g.t * g.e, st);
  cudaMemsetAsync(b.dell, 0, sizeof(float) * g.ns * g.t, st);
  cudaMemsetAsync(b.dellend, 0, sizeof(float) * g.ns * g.n, st);
  cudaMemsetAsync(b.dlam, 0, sizeof(float) * g.ns * g.n, st);
  int launches = 0;
  k_bwd_prep<T><<<nblk((size_t)g.ns * g.t, 256), 256, 0, st>>>(g, dy, w.y32, rowsum, b.dz);
  ++launches;
  if (tc4_supported(g, g.dtype)) {
    // degree 4 on the tensor cores (pa_tc4.cu): dA (feature-major GEMM), the
    // query- and update-side state VJPs (dphi GEMM + expand-VJP) and dv
    if (g.n > 1) {
      if (int rc = tc4_state(g, true, q, nullptr, b.dz, w.ell, w.lamlog, w.idx, w.wt, w.tc4, b.dA, st)) return rc;
      if (int rc = tc4_vjp(g, false, q, b.dq32, b.dell, nullptr, w.tc4, st)) return rc;
    }
    // reverse discumsum + fp16 operands of the state cotangents in one pass
    if (g.n == 1) cudaMemsetAsync(tc4_mxs(g, w.tc4), 0, sizeof(unsigned) * g.ns, st);
    if (int rc = tc4_scan_bwd(g, w.lamlog, w.A, b.dA, b.dlam, w.wt, w.tc4, st)) return rc;
    if (int rc = tc4_vjp(g, true, k, b.dk32, b.dell, b.dellend, w.tc4, st)) return rc;
    if (int rc = tc4_tok(g, 1, k, w.ell, w.lamlog, nullptr, nullptr, nullptr, nullptr, nullptr, b.dv32, w.tc4, st))
      return rc;
  } else {
  if (g.n > 1) {
    k_query_bwd<T, DM><<<dim3((g.n - 1) * ((g.c + ub_tokens<DM>() - 1) / ub_tokens<DM>()), g.ns), ub_tokens<DM>(),
                          dyn_smem(k_query_bwd<T, DM>, smb_query_bwd<DM>()), st>>>(g, q, w.A, w.idx, w.wt, w.ell, b.dz, b.dq32, b.dell);
    Geo gz = g;
    if (tc4_supported(g, g.dtype)) {
      if (int rc = tc4_state(g, true, q, nullptr, b.dz, w.ell, w.lamlog, w.idx, w.wt, w.tc4, b.dA, st)) return rc;
    } else if constexpr (DM <= 64)
      k_state_accum_f<T, float, DM><<<dim3((g.D + kSaThreads - 1) / kSaThreads, g.n - 1, g.ns), kSaThreads, 0, st>>>(
          gz, q, g.scale, g.gated ? 2 : 0, w.ell, w.lamlog, b.dz, 0, g.E1, g.E1, 0, w.idx, w.wt, 1, 1, b.dA);
    else
      k_state_accum<T, float, DM><<<dim3((g.D + 31) / 32, g.n - 1, g.ns), 256, 0, st>>>(
          gz, q, g.scale, g.gated ? 2 : 0, w.ell, w.lamlog, b.dz, 0, g.E1, g.E1, 0, w.idx, w.wt, 1, 1, b.dA);
    k_discumsum_bwd<<<dim3((unsigned)((per + 255) / 256), g.ns), 256, 0, st>>>(g, w.lamlog, w.A, b.dA, b.dlam);
    launches += 3;
  }
  k_update_bwd<T, DM><<<dim3(g.n * ((g.c + ub_tokens<DM>() - 1) / ub_tokens<DM>()), g.ns), ub_tokens<DM>(),
                        dyn_smem(k_update_bwd<T, DM>, smb_update_bwd<DM>()), st>>>(g, k, v, b.dA, w.idx, w.wt, w.ell, w.lamlog, b.dk32, b.dv32, b.dell, b.dellend);
  ++launches;
  }
  int intra_rc = 1;
  if (tc4_supported(g, g.dtype) && !getenv_flag("PA_TC4_INTRA_BWD_OFF")) {
    intra_rc = tc4_intra_bwd(g, w.ell, b.dz, dy, rowsum, b.dq32, b.dk32, b.dv32, b.dell, w.tc4, st);
    if (intra_rc > 1) return intra_rc;
  }
  if (intra_rc == 0) {
  } else if (DM == 32 && g.d == 32 && g.e == 32) {
    k_intra_bwd_q_h<T, kIntraTpr><<<dim3(g.n * tpc, g.ns), 64 * kIntraTpr, 0, st>>>(g, q, k, v, w.ell, b.dz, b.dq32,
                                                                                  b.dell);
    k_intra_bwd_kv_h<T, kIntraTpr><<<dim3(g.n * tpc, g.ns), 64 * kIntraTpr, 0, st>>>(g, q, k, v, w.ell, b.dz, b.dk32,
                                                                                   b.dv32, b.dell);
  } else {
    k_intra_bwd_q<T, DM><<<dim3(g.n * tpc, g.ns), 64, dyn_smem(k_intra_bwd_q<T, DM>, smb_intra_bwd<DM>()), st>>>(g, q, k, v, w.ell, b.dz, b.dq32, b.dell);
    k_intra_bwd_kv<T, DM><<<dim3(g.n * tpc, g.ns), 64, dyn_smem(k_intra_bwd_kv<T, DM>, smb_intra_bwd<DM>()), st>>>(g, q, k, v, w.ell, b.dz, b.dk32, b.dv32, b.dell);
  }
  launches += 3;
  if (dlogg) {
    k_gate_finish<<<(g.ns * g.n + 127) / 128, 128, 0, st>>>(g, w.lamlog, b.dell, b.dellend, b.dlam, dlogg);
    ++launches;
  }
  k_finalize<T><<<nblk((size_t)g.ns * g.t * g.d, 256), 256, 0, st>>>(g, b.dq32, g.d, dq);
  k_finalize<T><<<nblk((size_t)g.ns * g.t * g.d, 256), 256, 0, st>>>(g, b.dk32, g.d, dk);
  k_finalize<T><<<nblk((size_t)g.ns * g.t * g.e, 256), 256, 0, st>>>(g, b.dv32, g.e, dv);
  launches += 3;
  count_launch(launches);
  return cuda_check("simt backward");
}

template <typename T>
static int simt_forward_dm(const Geo& g, const void* q, const void* k, const void* v, const float* lg,
                           void* y, float* rs, const SimtWs& w, cudaStream_t st) {
  const int mx = std::max(g.d, g.e);
  if (mx <= 32)  // d = e = 32 (configs[2]): half the register rows and FMAs of DM = 64
    return simt_forward_t<T, 32>(g, (const T*)q, (const T*)k, (const T*)v, lg, (T*)y, rs, w, st);
  if (mx <= 64)
    return simt_forward_t<T, 64>(g, (const T*)q, (const T*)k, (const T*)v, lg, (T*)y, rs, w, st);
  return simt_forward_t<T, 128>(g, (const T*)q, (const T*)k, (const T*)v, lg, (T*)y, rs, w, st);
}

int simt_forward(const Geo& g, int dtype, const void* q, const void* k, const void* v, const float* lg,
                 void* y, float* rs, const SimtWs& w, cudaStream_t st) {
  switch (dtype) {
    case 0: return simt_forward_dm<float>(g, q, k, v, lg, y, rs, w, st);
    case 1: return simt_forward_dm<__nv_bfloat16>(g, q, k, v, lg, y, rs, w, st);
    case 2: return simt_forward_dm<__half>(g, q, k, v, lg, y, rs, w, st);
  }
  set_error("unsupported dtype for power_full");
  return 4;
}

template <typename T>
static int simt_backward_dm(const Geo& g, const void* q, const void* k, const void* v, const void* y,
                            const float* rs, const void* dy, void* dq, void* dk, void* dv,
                            float* dlogg, const SimtWs& w, const SimtBwdWs& b, cudaStream_t st) {
  const int mx = std::max(g.d, g.e);
  if (mx <= 32)
    return simt_backward_t<T, 32>(g, (const T*)q, (const T*)k, (const T*)v, (const T*)y, rs, (const T*)dy,
                                  (T*)dq, (T*)dk, (T*)dv, dlogg, w, b, st);
  if (mx <= 64)
    return simt_backward_t<T, 64>(g, (const T*)q, (const T*)k, (const T*)v, (const T*)y, rs, (const T*)dy,
                                  (T*)dq, (T*)dk, (T*)dv, dlogg, w, b, st);
  return simt_backward_t<T, 128>(g, (const T*)q, (const T*)k, (const T*)v, (const T*)y, rs, (const T*)dy,
                                 (T*)dq, (T*)dk, (T*)dv, dlogg, w, b, st);
}

int simt_backward(const Geo& g, int dtype, const void* q, const void* k, const void* v, const void* y,
                  const float* rs, const void* dy, void* dq, void* dk, void* dv, float* dlogg,
                  const SimtWs& w, const SimtBwdWs& b, cudaStream_t st) {
  switch (dtype) {
    case 0: return simt_backward_dm<float>(g, q, k, v, y, rs, dy, dq, dk, dv, dlogg, w, b, st);
    case 1: return simt_backward_dm<__nv_bfloat16>(g, q, k, v, y, rs, dy, dq, dk, dv, dlogg, w, b, st);
    case 2: return simt_backward_dm<__half>(g, q, k, v, y, rs, dy, dq, dk, dv, dlogg, w, b, st);
  }
  set_error("unsupported dtype for power_full backward");
  return 4;
}

int pub_update(int n, int c, int d, int e, int p, int D, int dtype, const void* k, const void* v,
               const void* w, const int* idx, const double* wt, void* state, void* ks, int acc,
               cudaStream_t st) {
  const size_t tot = (size_t)n * D * (e + 1);
  if (dtype == 3)
    k_pub_update<double><<<nblk(tot, 128), 128, 0, st>>>(n, c, d, e, p, D, (const double*)k, (const double*)v,
                                                         (const double*)w, idx, wt, (double*)state, (double*)ks, acc);
  else
    k_pub_update<float><<<nblk(tot, 128), 128, 0, st>>>(n, c, d, e, p, D, (const float*)k, (const float*)v,
                                                        (const float*)w, idx, wt, (float*)state, (float*)ks, acc);
  count_launch();
  return cuda_check("update_state");
}

int pub_query(int n, int c, int d, int e, int p, int D, int dtype, const void* q, const void* state,
              const void* ks, const int* idx, const double* wt, void* y, void* den, int acc, cudaStream_t st) {
  const size_t tot = (size_t)n * c * (e + 1);
  if (dtype == 3)
    k_pub_query<double><<<nblk(tot, 128), 128, 0, st>>>(n, c, d, e, p, D, (const double*)q, (const double*)state,
                                                        (const double*)ks, idx, wt, (double*)y, (double*)den, acc);
  else
    k_pub_query<float><<<nblk(tot, 128), 128, 0, st>>>(n, c, d, e, p, D, (const float*)q, (const float*)state,
                                                       (const float*)ks, idx, wt, (float*)y, (float*)den, acc);
  count_launch();
  return cuda_check("query_state");
}

int pub_discumsum(int n, int64_t L, int64_t M, int dtype, const void* values, const void* lams, void* out,
                  cudaStream_t st) {
  const size_t tot = (size_t)L * M;
  if (dtype == 3)
    k_pub_discumsum<double><<<nblk(tot, 256), 256, 0, st>>>(n, L, M, (const double*)values, (const double*)lams, (double*)out);
  else
    k_pub_discumsum<float><<<nblk(tot, 256), 256, 0, st>>>(n, L, M, (const float*)values, (const float*)lams, (float*)out);
  count_launch();
  return cuda_check("discumsum");
}

}  // namespace pa

namespace pa {
int64_t host_binom(int64_t n, int64_t k) { return binom(n, k); }

// pieces reused by the bf16 tensor-core backward (pa_tc.cu)
int simt_intra_bwd(const Geo& g, const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                   const float* ell, const float* dz, float* dq32, float* dk32, float* dv32, float* dell,
                   cudaStream_t st) {
  using T = __nv_bfloat16;
  const int tpc = (g.c + 63) / 64;
  k_intra_bwd_q<T, 64><<<dim3(g.n * tpc, g.ns), 64, dyn_smem(k_intra_bwd_q<T, 64>, smb_intra_bwd<64>()), st>>>(
      g, q, k, v, ell, dz, dq32, dell);
  k_intra_bwd_kv<T, 64><<<dim3(g.n * tpc, g.ns), 64, dyn_smem(k_intra_bwd_kv<T, 64>, smb_intra_bwd<64>()), st>>>(
      g, q, k, v, ell, dz, dk32, dv32, dell);
  count_launch(2);
  return cuda_check("intra backward");
}

int simt_gate_finish(const Geo& g, const float* lamlog, const float* dell, const float* dellend,
                     const float* dlam, float* dlogg, cudaStream_t st) {
  k_gate_finish<<<(g.ns * g.n + 127) / 128, 128, 0, st>>>(g, lamlog, dell, dellend, dlam, dlogg);
  count_launch();
  return cuda_check("gate finish");
}

int simt_finalize_bf16(const Geo& g, const float* src, int w, void* dst, cudaStream_t st) {
  k_finalize<__nv_bfloat16><<<nblk((size_t)g.ns * g.t * w, 256), 256, 0, st>>>(g, src, w, (__nv_bfloat16*)dst);
  count_launch();
  return cuda_check("finalize");
}
}  // namespace pa
