// bf16 tcgen05 pipeline for SPOW p = 2, d = e = 64 (the north-star shape).
//
// Forward (per stream s, chunk k; reference chunked.py:287-413):
//   prep_gates : ell = in-chunk cumsum of log g, lamlog = ell at chunk end
//   prep_kt    : K~^T [dim][token] with k~_j = k_j * exp((ell_end - ell_j)/2),
//                so phi'(k~_j) = W_j phi'(k_j) (suffix decay, chunked.py:89-95)
//   upd        : S'_k = phi'(K~)^T [V | 1] -- tcgen05, A = phi'(K~)^T generated
//                into TMEM from K~^T in smem (update_state, kernels.py:55-83)
//   scan       : A'_k = lambda_k A'_{k-1} + omega * S'_k in fp32 (discumsum,
//                chunked.py:156-176), stored bf16 in the compact [u][f] tiles
//   out        : y = intra-chunk power attention (S = Q K^T, P = decay * s^2,
//                O += P V on tcgen05) + phi'(q~) A'_{k-1} with phi'(q~)
//                generated from registers into TMEM (query_state + combine,
//                chunked.py:372-395); one TMEM accumulator for both.
#include <cuda.h>

#include <stdio.h>

#include <algorithm>
#include <utility>
#include <vector>

#include "pa_common.cuh"
#include "pa_simt.cuh"
#include "pa_sm100.cuh"
#include "pa_tc.cuh"
#include "pa_tc_common.cuh"

namespace pa {
using namespace sm100;
using namespace tc;

__constant__ BlkTab c_blk = make_blk_tab();

// ==========================================================================
// prep kernels
// ==========================================================================
// one warp per (stream, chunk): inclusive scan of log g over the chunk
__global__ void __launch_bounds__(128) k_tc_prep_gates(Geo g, const float* __restrict__ log_g, float* ell,
                                                       float* lamlog) {
  const int wid = (blockIdx.x * 4) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (wid >= g.ns * g.n) return;
  const int s = wid / g.n, k = wid - s * g.n;
  const int s0 = k * g.c, s1 = min(s0 + g.c, g.t);
  float carry = 0.f;
  for (int m0 = s0; m0 < s1; m0 += 32) {
    const int m = m0 + lane;
    float x = (m < s1 && g.gated) ? fmaxf(log_g[rowid(g, s, m)], -80.f) : 0.f;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      float y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    x += carry;
    if (m < s1) ell[(size_t)s * g.t + m] = x;
    carry = __shfl_sync(0xffffffffu, x, 31);
  }
  if (lane == 0) lamlog[wid] = carry;
}

// X~^T [((s*n + k)*64 + dim)][tok] = x_j * exp(mode) for 64-token blocks;
// mode 0: exp((lend - ell_j)/2) (keys, suffix decay); 1: scale*exp(ell_j/2) (queries, prefix)
__global__ void __launch_bounds__(256) k_tc_prep_xt(Geo g, const __nv_bfloat16* __restrict__ x,
                                                    const float* __restrict__ ell,
                                                    const float* __restrict__ lamlog, int mode,
                                                    __nv_bfloat16* xt) {
  __shared__ float tile[64][65];
  const int tb = blockIdx.x, k = blockIdx.y, s = blockIdx.z;
  const int j0 = k * g.c + tb * 64;
  // load 64 tokens x 64 dims (coalesced rows), scale per token
  for (int i = threadIdx.x; i < 64 * 64; i += 256) {
    const int r = i >> 6, dcol = i & 63;
    const int j = j0 + r;
    const float lj = ell[(size_t)s * g.t + j];
    const float f = mode == 0 ? __expf(0.5f * (lamlog[s * g.n + k] - lj)) : g.scale * __expf(0.5f * lj);
    tile[r][dcol] = __bfloat162float(x[rowid(g, s, j) * HD + dcol]) * (g.gated || mode ? f : 1.f);
  }
  __syncthreads();
  __nv_bfloat16* dst = xt + ((size_t)(s * g.n + k) * HD) * g.c + tb * 64;
  for (int i = threadIdx.x; i < 64 * 64; i += 256) {
    const int dim = i >> 6, r = i & 63;
    dst[(size_t)dim * g.c + r] = __float2bfloat16_rn(tile[r][dim]);
  }
}

// ==========================================================================
// feature-major GEMM ("hard shape"): M = 128-row tiles of block-order
// features, K = tokens of one chunk, A = phi'(X~)^T generated into TMEM from
// X~^T tiles, B = per-token rows (MN-major) + a 16-column score-sum block.
//   forward  (update_state, kernels.py:55-83):  X~ = K~, B = [V | 1]     -> S'_k
//   backward (query_state VJP, gradients.py:429-430): X~ = Q~, B = [dnum | dden] -> dA'_{k-1}
// Warp roles (256 threads): w0 TMA producer, w1 MMA issuer, w2 TMEM owner,
// w4..w7 generate A (lane quadrant = warp % 4) and run the epilogue.
// grid (group of 4 tiles, chunk, stream)
// ==========================================================================
namespace fm {
constexpr int ST = 4;                 // 64-token TMA stages
constexpr int NB = 3;                 // TMEM A buffers (32 tokens each)
constexpr int TOK = 64;
constexpr int XT_B = 64 * 128;        // 64 dims x 64 tokens bf16
constexpr int B_B = 64 * 128;         // 64 tokens x 64 values bf16
constexpr int B16_B = 64 * 32;        // 64 tokens x 16 bf16 (SW32)
constexpr int SMEM_USED = 1024 + ST * (XT_B + B_B + B16_B) + 2048 + 512;
constexpr int SMEM = SMEM_USED > 120 * 1024 ? SMEM_USED : 120 * 1024;  // 1 CTA (512 TMEM cols) per SM
}  // namespace fm

template <bool kBwd>
__global__ void __launch_bounds__(256, 1) k_tc_featmajor(const __grid_constant__ CUtensorMap tm_xt,
                                                         const __grid_constant__ CUtensorMap tm_b,
                                                         const __grid_constant__ CUtensorMap tm_b16, Geo g,
                                                         int with_den, float* out) {
  using namespace fm;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keep the shared address space
  uint8_t* xt_s = smem;
  uint8_t* b_s = xt_s + ST * XT_B;
  uint8_t* b16_s = b_s + ST * B_B;
  uint8_t* ones = b16_s + ST * B16_B;
  uint64_t* bars = (uint64_t*)(ones + 2048);
  uint64_t* full = bars;                 // [ST]
  uint64_t* empty = bars + ST;           // [ST]
  uint64_t* afull = bars + 2 * ST;       // [NB]
  uint64_t* aempty = afull + NB;         // [NB]
  uint64_t* fin = aempty + NB;           // [1]
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int grp = blockIdx.x, kin = blockIdx.y + (kBwd ? 1 : 0), s = blockIdx.z;
  const int slot = kBwd ? kin - 1 : kin;
  const int t0 = grp * 4, nt = min(4, NTH - t0);
  const int nsub = g.c / 32, nstage = g.c / TOK;
  const bool den = with_den != 0;

  if (w == 2) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    for (int i = 0; i < ST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < NB; ++i) {
      mbar_init(&afull[i], 4);
      mbar_init(&aempty[i], 1);
    }
    mbar_init(fin, 1);
    fence_barrier_init();
  }
  if (!kBwd)  // K-major 16-row block whose row 0 is all ones: the key_sum column
    for (int i = tid; i < 2048 / 4; i += 256) ((uint32_t*)ones)[i] = (i < 32) ? 0x3F803F80u : 0u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;

  if (w == 0) {
    // ---------------- producer ----------------
    if (l == 0) {
      tma_prefetch(&tm_xt);
      tma_prefetch(&tm_b);
      const int row0 = (s * g.n + kin) * HD;
      const int bi = s / g.h, hi = s % g.h;
      for (int j = 0; j < nstage; ++j) {
        const int st = j % ST;
        if (j >= ST) mbar_wait(&empty[st], ((j / ST) + 1) & 1);
        const uint32_t bytes = XT_B + B_B + ((kBwd && den) ? B16_B : 0);
        mbar_expect_tx(&full[st], bytes);
        tma_load_2d(xt_s + st * XT_B, &tm_xt, &full[st], j * TOK, row0);
        if (kBwd) {
          tma_load_2d(b_s + st * B_B, &tm_b, &full[st], 0, s * g.t + kin * g.c + j * TOK);
          if (den) tma_load_2d(b16_s + st * B16_B, &tm_b16, &full[st], 0, s * g.t + kin * g.c + j * TOK);
        } else {
          tma_load_4d(b_s + st * B_B, &tm_b, &full[st], 0, hi, kin * g.c + j * TOK, bi);
        }
      }
    }
  } else if (w == 1) {
    // ---------------- MMA issuer ----------------
    if (l == 0) {
      const uint32_t id64 = idesc_bf16(128, 64, false, true);
      const uint32_t id16 = idesc_bf16(128, 16, false, !kBwd ? false : true);
      for (int i = 0; i < nsub; ++i) {
        const int j = i >> 1, h = i & 1, st = j % ST, buf = i % NB;
        mbar_wait(&full[st], (j / ST) & 1);
        mbar_wait(&afull[buf], (i / NB) & 1);
        tc_fence_after();
        const uint32_t bsm = smem_u32(b_s + st * B_B);
        const uint32_t b16 = smem_u32(b16_s + st * B16_B);
        for (int t = 0; t < nt; ++t) {
          const uint32_t acc = tm + (uint32_t)(t * UW);
          const uint32_t ab = tm + 320u + (uint32_t)((buf * 4 + t) * 16);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const uint32_t f = (i > 0 || kk > 0) ? 1u : 0u;
            const int trow = h * 32 + kk * 16;  // token row inside the 64-token stage
            mma_ts(acc, ab + kk * 8, smem_desc(bsm + trow * 128, 8192, 1024, 2), id64, f);
            if (den) {
              const uint64_t dd = kBwd ? smem_desc(b16 + trow * 32, 512, 256, 6)
                                       : smem_desc(smem_u32(ones) + ((h * 2 + kk) & 3) * 32, 16, 1024, 2);
              mma_ts(acc + 64, ab + kk * 8, dd, id16, f);
            }
          }
        }
        tc_commit(&aempty[buf]);
        if (h == 1) tc_commit(&empty[st]);
      }
      tc_commit(fin);
    }
  } else if (w >= 4) {
    // ---------------- A generation (phi'(X~)^T into TMEM) ----------------
    const int q = w & 3;
    int ra[4], rb[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int blk = (t < nt) ? (t0 + t) * 4 + q : 0;
      ra[t] = 4 * c_blk.al[blk] + (l >> 3);
      rb[t] = 8 * c_blk.be[blk] + (l & 7);
    }
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    for (int i = 0; i < nsub; ++i) {
      const int j = i >> 1, h = i & 1, st = j % ST, buf = i % NB;
      mbar_wait(&full[st], (j / ST) & 1);
      if (i >= NB) mbar_wait(&aempty[buf], ((i / NB) + 1) & 1);
      const uint8_t* xs = xt_s + st * XT_B;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (t < nt) {
          uint32_t va[16], vb[16], o[16];
#pragma unroll
          for (int c4 = 0; c4 < 4; ++c4) {
            const int ch = h * 4 + c4;
            *(uint4*)&va[c4 * 4] = *(const uint4*)(xs + sw128_off(ra[t], ch));
            *(uint4*)&vb[c4 * 4] = *(const uint4*)(xs + sw128_off(rb[t], ch));
          }
#pragma unroll
          for (int c = 0; c < 16; ++c) o[c] = hmul2_bf16(va[c], vb[c]);
          tmem_st16(tm + 320u + (uint32_t)((buf * 4 + t) * 16) + lane_off, o);
        }
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (l == 0) mbar_arrive(&afull[buf]);
    }
    // ---------------- epilogue ----------------
    mbar_wait(fin, 0);
    tc_fence_after();
    const int ncols = den ? UW : 64;
    for (int t = 0; t < nt; ++t) {
      float* dst = out + (((size_t)(s * g.n + slot) * FH) + (size_t)(t0 + t) * 128 + q * 32 + l) * UW;
      for (int c0 = 0; c0 < ncols; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(tm + (uint32_t)(t * UW) + lane_off + c0, r);
        tc_wait_ld();
#pragma unroll
        for (int c = 0; c < 16; c += 4)
          *(float4*)(dst + c0 + c) = make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]),
                                                 __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 2) tmem_dealloc<512>(tm);
}

// ==========================================================================
// scan (discumsum over chunk states) + reorder to compact [u][f] bf16 tiles
//   A'_k = lambda_k A'_{k-1} + omega_f S'_k      (chunked.py:156-176, 356-367)
// grid (33 feature blocks, stream); 256 threads
// ==========================================================================
__device__ __forceinline__ int hard_slot(int a, int b) {
  const int blk = c_blk.idx[a >> 2][b >> 3];
  return blk * 32 + (a & 3) * 8 + (b & 7);
}

__device__ __forceinline__ uint32_t st_off(int u, int f) {  // byte offset inside a [80][64] bf16 tile
  return (uint32_t)u * 128u + ((((uint32_t)f >> 3) ^ ((uint32_t)u & 7u)) << 4) + ((uint32_t)f & 7u) * 2u;
}

__global__ void __launch_bounds__(256) k_tc_scan_fwd(Geo g, int ucols, const float* __restrict__ lamlog,
                                                     const float* __restrict__ sp, __nv_bfloat16* stout) {
  __shared__ float tile[64][UW + 1];
  __shared__ int rows[64];
  __shared__ float om[64];
  const int fb = blockIdx.x, s = blockIdx.y, tid = threadIdx.x;
  if (tid < 64) {
    int a, b;
    compact_ab(fb * 64 + tid, a, b);
    rows[tid] = (a <= b) ? hard_slot(a, b) : -1;
    om[tid] = (a == b) ? 1.f : (a < b ? 2.f : 0.f);
  }
  __syncthreads();
  const int fl = tid & 63, u0 = tid >> 6;
  constexpr int PER = UW / 4;  // 20 columns per thread
  float acc[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) acc[i] = 0.f;
  for (int k = 0; k < g.n; ++k) {
    __syncthreads();
    const float* src = sp + (size_t)(s * g.n + k) * FH * UW;
    for (int i = tid; i < 64 * UW; i += 256) {
      const int r = i / UW, u = i - r * UW;
      tile[r][u] = (rows[r] >= 0 && u < ucols) ? src[(size_t)rows[r] * UW + u] : 0.f;
    }
    __syncthreads();
    const float lam = (k == 0 || !g.gated) ? (k == 0 ? 0.f : 1.f) : __expf(lamlog[s * g.n + k]);
    uint8_t* dst = (uint8_t*)(stout + ((size_t)(s * g.n + k) * NFB + fb) * (UW * 64));
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int u = u0 + 4 * i;
      acc[i] = lam * acc[i] + om[fl] * tile[fl][u];
      *(__nv_bfloat16*)(dst + st_off(u, fl)) = __float2bfloat16_rn(acc[i]);
    }
  }
}

// ==========================================================================
// out: fused intra-chunk power attention + state query + combine + normalize
// (attention.py:273-309 per chunk, kernels.py:86-110, chunked.py:372-395)
// Warp roles (256 threads): w0 loads (TMA Q/K/V, bulk state blocks), w1 MMA
// issuer, w2 TMEM owner, w4..w7 compute (phi'(q~) generation, P = decay*s^2,
// epilogue).  TMEM: O [0,80), A buffers [128,256), S/P buffers [256,512).
// grid (query tile of 128, chunk, stream)
// ==========================================================================
namespace outk {
constexpr int QB = 128 * 128;           // Q tile bytes (128 tok x 64 dims bf16)
constexpr int KB = 128 * 128;           // K tile
constexpr int VB = 128 * 128;           // V tile
constexpr int STB = UW * 128;           // state block (80 u x 64 f bf16)
constexpr int KV_ST = 3;
constexpr int ST_ST = 8;
constexpr int NA = 4;                   // TMEM A buffers (64 features each)
constexpr int SMEM = 1024 + QB + KV_ST * (KB + VB) + ST_ST * STB + 2048 + 4096 + 1024 + 512;
}  // namespace outk

template <int C>
__device__ __forceinline__ uint32_t bcast_a(const uint32_t* qp) {
  constexpr int a = col_a(C);
  return __byte_perm(qp[a >> 1], 0, (a & 1) ? 0x3232 : 0x1010);
}
template <int FB, int... I>
__device__ __forceinline__ void gen_block(const uint32_t* qp, uint32_t* o, std::integer_sequence<int, I...>) {
  ((o[I] = hmul2_bf16(bcast_a<FB * 32 + I>(qp), qp[col_beta(FB * 32 + I)])), ...);
}

// compute warps: phi'(x) for the 33 compact feature blocks of one token row,
// each written to a TMEM A buffer and handed to the MMA warp via a_full.
template <int FB>
__device__ __forceinline__ void gen_all_blocks(const uint32_t (&qp)[32], uint32_t a_base, uint32_t lane_off,
                                               uint64_t* a_full, uint64_t* a_empty, int l) {
  constexpr int NA = outk::NA;
  constexpr int bb = FB % NA;
  if (FB >= NA) mbar_wait(&a_empty[bb], ((FB / NA) + 1) & 1);
  uint32_t o[32];
  gen_block<FB>(qp, o, std::make_integer_sequence<int, 32>{});
  const uint32_t ast = a_base + (uint32_t)(bb * 32) + lane_off;
  tmem_st16(ast, o);
  tmem_st16(ast + 16, o + 16);
  tc_wait_st();
  tc_fence_before();
  __syncwarp();
  if (l == 0) mbar_arrive(&a_full[bb]);
  if constexpr (FB + 1 < NFB) gen_all_blocks<FB + 1>(qp, a_base, lane_off, a_full, a_empty, l);
}

__global__ void __launch_bounds__(256, 1) k_tc_out(const __grid_constant__ CUtensorMap tm_q,
                                                   const __grid_constant__ CUtensorMap tm_k,
                                                   const __grid_constant__ CUtensorMap tm_v, Geo g,
                                                   const __nv_bfloat16* __restrict__ qraw,
                                                   const float* __restrict__ ell,
                                                   const __nv_bfloat16* __restrict__ st_all, int with_den,
                                                   __nv_bfloat16* y, float* rowsum, float* y32, int* zflag,
                                                   unsigned long long* dbg) {
  using namespace outk;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // keep the shared address space
  uint8_t* q_s = smem;
  uint8_t* k_s = q_s + QB;
  uint8_t* v_s = k_s + KV_ST * KB;
  uint8_t* st_s = v_s + KV_ST * VB;
  uint8_t* ones = st_s + ST_ST * STB;
  float* ell_s = (float*)(ones + 2048);       // [1024]
  float* cj = ell_s + 1024;                   // [2][128]
  uint64_t* bars = (uint64_t*)(cj + 256);
  uint64_t* q_full = bars;                    // 1
  uint64_t* kv_full = q_full + 1;             // KV_ST
  uint64_t* kv_empty = kv_full + KV_ST;       // KV_ST
  uint64_t* st_full = kv_empty + KV_ST;       // ST_ST
  uint64_t* st_empty = st_full + ST_ST;       // ST_ST
  uint64_t* a_full = st_empty + ST_ST;        // NA
  uint64_t* a_empty = a_full + NA;            // NA
  uint64_t* s_full = a_empty + NA;            // 2
  uint64_t* p_full = s_full + 2;              // 2
  uint64_t* pv_done = p_full + 2;             // 2
  uint64_t* fin = pv_done + 2;                // 1
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int I = blockIdx.x, k = blockIdx.y, s = blockIdx.z;
  const int bi = s / g.h, hi = s % g.h;
  const int c0 = k * g.c;
  const bool den = with_den != 0;
  const bool has_state = k >= 1;

  if (w == 2) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < KV_ST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < ST_ST; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], 1);
    }
    for (int i = 0; i < NA; ++i) {
      mbar_init(&a_full[i], 4);
      mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(fin, 1);
    fence_barrier_init();
  }
  for (int i = tid; i < 2048 / 4; i += 256) ((uint32_t*)ones)[i] = (i < 32) ? 0x3F803F80u : 0u;
  for (int i = tid; i < g.c; i += 256) ell_s[i] = ell[(size_t)s * g.t + c0 + i];
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  const uint32_t a_base = tm + 128u;
  auto sbuf = [&](int b) { return tm + 256u + (uint32_t)(b * 128); };
  const size_t cta = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
  auto stamp = [&](int i) {
    if (dbg) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      dbg[cta * 64 + i] = t;
    }
  };
  if (tid == 0) stamp(0);

  if (w == 0) {
    // ---------------- loads ----------------
    if (l == 0) {
      tma_prefetch(&tm_q);
      tma_prefetch(&tm_k);
      tma_prefetch(&tm_v);
      mbar_expect_tx(q_full, QB);
      tma_load_4d(q_s, &tm_q, q_full, 0, hi, c0 + I * 128, bi);
      auto kv = [&](int J) {
        const int st = J % KV_ST;
        if (J >= KV_ST) mbar_wait(&kv_empty[st], ((J / KV_ST) + 1) & 1);
        if (J < 8) stamp(8 + J);
        mbar_expect_tx(&kv_full[st], KB + VB);
        tma_load_4d(k_s + st * KB, &tm_k, &kv_full[st], 0, hi, c0 + J * 128, bi);
        tma_load_4d(v_s + st * VB, &tm_v, &kv_full[st], 0, hi, c0 + J * 128, bi);
      };
      const int early = min(I + 1, KV_ST);
      for (int J = 0; J < early; ++J) kv(J);
      if (has_state) {
        const __nv_bfloat16* src = st_all + ((size_t)(s * g.n + (k - 1)) * NFB) * (UW * 64);
        const uint32_t bytes = den ? STB : 64 * 128;
        for (int fb = 0; fb < NFB; ++fb) {
          const int sb = fb % ST_ST;
          if (fb >= ST_ST) mbar_wait(&st_empty[sb], ((fb / ST_ST) + 1) & 1);
          mbar_expect_tx(&st_full[sb], bytes);
          bulk_load(st_s + sb * STB, src + (size_t)fb * (UW * 64), bytes, &st_full[sb]);
        }
      }
      for (int J = early; J <= I; ++J) kv(J);
    }
  } else if (w == 1) {
    // ---------------- MMA issuer ----------------
    if (l == 0) {
      const uint32_t id64k = idesc_bf16(128, 64, false, false);
      const uint32_t id16k = idesc_bf16(128, 16, false, false);
      const uint32_t id64mn = idesc_bf16(128, 64, false, true);
      const uint32_t id128 = idesc_bf16(128, 128, false, false);
      if (has_state) {
        for (int fb = 0; fb < NFB; ++fb) {
          const int bb = fb % NA, sb = fb % ST_ST;
          mbar_wait(&a_full[bb], (fb / NA) & 1);
          mbar_wait(&st_full[sb], (fb / ST_ST) & 1);
          tc_fence_after();
          const uint32_t sbase = smem_u32(st_s + sb * STB);
          const uint32_t ab = a_base + (uint32_t)(bb * 32);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t f = (fb > 0 || kk > 0) ? 1u : 0u;
            mma_ts(tm, ab + kk * 8, smem_desc(sbase + kk * 32, 16, 1024, 2), id64k, f);
            if (den) mma_ts(tm + 64, ab + kk * 8, smem_desc(sbase + 8192 + kk * 32, 16, 1024, 2), id16k, f);
          }
          tc_commit(&a_empty[bb]);
          tc_commit(&st_empty[sb]);
        }
      }
      stamp(1);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int J) {
        const int st = J % KV_ST, sb = J & 1;
        mbar_wait(&kv_full[st], (J / KV_ST) & 1);
        if (J >= 2) mbar_wait(&pv_done[sb], ((J >> 1) + 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ss(sbuf(sb), smem_desc(smem_u32(q_s) + kk * 32, 16, 1024, 2),
                 smem_desc(smem_u32(k_s + st * KB) + kk * 32, 16, 1024, 2), id128, kk > 0 ? 1u : 0u);
        tc_commit(&s_full[sb]);
        if (J < 8) stamp(16 + J);
      };
      issue_s(0);
      for (int J = 0; J <= I; ++J) {
        if (J + 1 <= I) issue_s(J + 1);
        const int sb = J & 1, st = J % KV_ST;
        mbar_wait(&p_full[sb], (J >> 1) & 1);
        if (J < 8) stamp(24 + J);
        tc_fence_after();
        const uint32_t vb = smem_u32(v_s + st * VB);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t f = (has_state || J > 0 || kk > 0) ? 1u : 0u;
          mma_ts(tm, sbuf(sb) + kk * 8, smem_desc(vb + kk * 2048, 8192, 1024, 2), id64mn, f);
          if (den)
            mma_ts(tm + 64, sbuf(sb) + kk * 8, smem_desc(smem_u32(ones) + (kk & 3) * 32, 16, 1024, 2), id16k, f);
        }
        tc_commit(&pv_done[sb]);
        tc_commit(&kv_empty[st]);
      }
      tc_commit(fin);
      stamp(2);
    }
  } else if (w >= 4) {
    // ---------------- compute warps ----------------
    const int q = w & 3, row = q * 32 + l;      // TMEM lane == query row in the tile
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int tok = c0 + I * 128 + row;
    const float li = ell_s[I * 128 + row];
    const float sig2 = g.scale * g.scale;
    if (has_state) {
      uint32_t qp[32];
      const float f = g.scale * __expf(0.5f * li);
      const uint4* qrow = (const uint4*)(qraw + rowid(g, s, tok) * HD);
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        uint4 v4 = qrow[c8];
        const uint32_t* pv = (const uint32_t*)&v4;
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2) {
          float2 f2 = __bfloat1622float2(*(const __nv_bfloat162*)&pv[e2]);
          qp[c8 * 4 + e2] = pack_bf16(f2.x * f, f2.y * f);
        }
      }
      gen_all_blocks<0>(qp, a_base, lane_off, a_full, a_empty, l);
    }
    if (tid == 128) stamp(3);
    for (int J = 0; J <= I; ++J) {
      const int sb = J & 1;
      const bool diag = (J == I);
      const float lref = ell_s[J * 128 + 127];
      cj[sb * 128 + row] = diag ? ell_s[J * 128 + row] : __expf(lref - ell_s[J * 128 + row]);
      asm volatile("bar.sync 1, 128;" ::: "memory");
      mbar_wait(&s_full[sb], (J >> 1) & 1);
      if (tid == 128 && J < 8) stamp(32 + J);
      tc_fence_after();
      const float ri = __expf(li - lref) * sig2;
      const float* cjs = cj + sb * 128;
      if (!diag) {
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t r[32], pk[16];
          tmem_ld32(sbuf(sb) + lane_off + ch * 32, r);
          tc_wait_ld();
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            const float4 c4 = *(const float4*)(cjs + ch * 32 + e4 * 4);
            const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
            for (int z = 0; z < 4; z += 2) {
              const float s0 = __uint_as_float(r[e4 * 4 + z]), s1 = __uint_as_float(r[e4 * 4 + z + 1]);
              pk[e4 * 2 + z / 2] = pack_bf16(ri * cc[z] * s0 * s0, ri * cc[z + 1] * s1 * s1);
            }
          }
          tmem_st16(sbuf(sb) + lane_off + ch * 16, pk);
        }
      } else {
        // diagonal block: exact pairwise decay exp(ell_i - ell_j), causal mask j <= i
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t r[32], pk[16];
          tmem_ld32(sbuf(sb) + lane_off + ch * 32, r);
          tc_wait_ld();
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            const float4 c4 = *(const float4*)(cjs + ch * 32 + e4 * 4);
            const float cc[4] = {c4.x, c4.y, c4.z, c4.w};
            float pv[4];
#pragma unroll
            for (int z = 0; z < 4; ++z) {
              const int jj = ch * 32 + e4 * 4 + z;
              const float sv = __uint_as_float(r[e4 * 4 + z]);
              const float e = __expf(fminf(li - cc[z], 0.f)) * sig2 * sv * sv;
              pv[z] = (jj <= row) ? e : 0.f;
            }
            pk[e4 * 2] = pack_bf16(pv[0], pv[1]);
            pk[e4 * 2 + 1] = pack_bf16(pv[2], pv[3]);
          }
          tmem_st16(sbuf(sb) + lane_off + ch * 16, pk);
        }
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (l == 0) mbar_arrive(&p_full[sb]);
      if (tid == 128 && J < 8) stamp(40 + J);
    }
    // ---------------- epilogue ----------------
    mbar_wait(fin, 0);
    tc_fence_after();
    uint32_t o[64];
    tmem_ld32(tm + lane_off, o);
    tmem_ld32(tm + lane_off + 32, o + 32);
    float dn = 0.f;
    if (den) {
      uint32_t r[16];
      tmem_ld16(tm + lane_off + 64, r);
      tc_wait_ld();
      dn = __uint_as_float(r[0]);
    }
    tc_wait_ld();
    const size_t rw = rowid(g, s, tok);
    float inv = 1.f;
    if (g.normalize) {
      if (!(dn > 0.f)) atomicAdd(zflag, 1);
      inv = 1.f / dn;
    }
    if (rowsum) rowsum[rw] = dn;
    uint4* yrow = (uint4*)(y + rw * HD);
#pragma unroll
    for (int c8 = 0; c8 < 8; ++c8) {
      uint4 v4;
      uint32_t* pv = (uint32_t*)&v4;
#pragma unroll
      for (int e2 = 0; e2 < 4; ++e2)
        pv[e2] = pack_bf16(__uint_as_float(o[c8 * 8 + e2 * 2]) * inv, __uint_as_float(o[c8 * 8 + e2 * 2 + 1]) * inv);
      yrow[c8] = v4;
    }
    if (g.normalize && y32) {
      float4* dst = (float4*)(y32 + ((size_t)s * g.t + tok) * HD);
#pragma unroll
      for (int c4 = 0; c4 < 16; ++c4)
        dst[c4] = make_float4(__uint_as_float(o[c4 * 4]) * inv, __uint_as_float(o[c4 * 4 + 1]) * inv,
                              __uint_as_float(o[c4 * 4 + 2]) * inv, __uint_as_float(o[c4 * 4 + 3]) * inv);
    }
  }
  if (tid == 128) stamp(6);
  tc_fence_before();
  __syncthreads();
  if (w == 2) tmem_dealloc<512>(tm);
}

// ==========================================================================
// host side
// ==========================================================================
struct TcFwdWs {
  int* zflag;
  float* ell;
  float* lamlog;
  __nv_bfloat16* kt;
  float* sp;
  __nv_bfloat16* st;
  float* y32;
};

static size_t a256(size_t x) { return (x + 255) & ~size_t(255); }

static TcFwdWs carve_fwd(const Geo& g, void* base, size_t* bytes) {
  char* p = (char*)base;
  size_t off = 0;
  auto take = [&](size_t n) {
    void* r = p ? p + off : nullptr;
    off += a256(n);
    return r;
  };
  TcFwdWs w;
  w.zflag = (int*)take(4);
  w.ell = (float*)take(sizeof(float) * g.ns * g.t);
  w.lamlog = (float*)take(sizeof(float) * g.ns * g.n);
  w.kt = (__nv_bfloat16*)take(2ull * g.ns * g.t * HD);
  w.sp = (float*)take(4ull * g.ns * g.n * FH * UW);
  w.st = (__nv_bfloat16*)take(2ull * g.ns * g.n * NFB * UW * 64);
  w.y32 = (float*)take(g.normalize ? 4ull * g.ns * g.t * HD : 0);
  *bytes = off;
  return w;
}

bool tc_supported(const Geo& g, int dtype) {
  static const bool disabled = [] {
    const char* e = getenv("PA_DISABLE_TC");
    return e && e[0] == '1';
  }();
  return !disabled && dtype == 1 && g.p == 2 && g.d == HD && g.e == HD && g.c % 128 == 0 && g.c <= 1024 &&
         g.t % g.c == 0;
}

size_t tc_fwd_workspace_bytes(const Geo& g) {
  size_t n;
  carve_fwd(g, nullptr, &n);
  return n;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point, so the
// library has no link-time dependency on libcuda (it loads on GPU-less hosts).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (EncodeTiledFn) nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}

static bool make_map_4d(CUtensorMap* m, const void* ptr, const Geo& g, int box_tokens) {
  // [b][t][h][64] bf16: dims inner -> outer {64, h, t, b}
  cuuint64_t dims[4] = {(cuuint64_t)HD, (cuuint64_t)g.h, (cuuint64_t)g.t, (cuuint64_t)g.b};
  cuuint64_t strides[3] = {(cuuint64_t)HD * 2, (cuuint64_t)g.h * HD * 2, (cuuint64_t)g.t * g.h * HD * 2};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)box_tokens, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return encode_fn() && encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box,
                                es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool make_map_xt(CUtensorMap* m, const void* ptr, const Geo& g) {
  // [ns*n*64 rows][c tokens] bf16, box 64 tokens x 64 rows
  cuuint64_t dims[2] = {(cuuint64_t)g.c, (cuuint64_t)g.ns * g.n * HD};
  cuuint64_t strides[1] = {(cuuint64_t)g.c * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t es[2] = {1, 1};
  return encode_fn() && encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                                es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// PA_DEBUG_TIMING=1: per-CTA globaltimer stamps of k_tc_out (investigation aid)
static unsigned long long* g_dbg = nullptr;
static size_t g_dbg_n = 0;
static unsigned long long* dbg_buf(const Geo& g) {
  static const bool on = [] {
    const char* e = getenv("PA_DEBUG_TIMING");
    return e && e[0] == '1';
  }();
  if (!on) return nullptr;
  size_t n = (size_t)(g.c / 128) * g.n * g.ns * 64;
  if (n > g_dbg_n) {
    if (g_dbg) cudaFree(g_dbg);
    cudaMalloc(&g_dbg, n * 8);
    g_dbg_n = n;
  }
  cudaMemset(g_dbg, 0, n * 8);
  return g_dbg;
}
static void dbg_report(const Geo& g, cudaStream_t st) {
  if (!g_dbg) return;
  cudaStreamSynchronize(st);
  size_t ncta = (size_t)(g.c / 128) * g.n * g.ns;
  std::vector<unsigned long long> h(ncta * 64);
  cudaMemcpy(h.data(), g_dbg, h.size() * 8, cudaMemcpyDeviceToHost);
  double acc[8] = {0};
  unsigned long long tmin = ~0ull, tmax = 0;
  for (size_t c = 0; c < ncta; ++c) {
    unsigned long long* r = &h[c * 64];
    tmin = std::min(tmin, r[0]);
    tmax = std::max(tmax, r[6]);
    for (int i = 1; i <= 6; ++i) acc[i] += (double)(r[i] - r[0]);
  }
  fprintf(stderr, "[k_tc_out] ctas %zu span %.3f ms; mean since start (us): mmaA_done %.2f fin_issued %.2f genA_done %.2f loopB_done %.2f fin_seen %.2f end %.2f\n",
          ncta, (tmax - tmin) * 1e-6, acc[1] / ncta * 1e-3, acc[2] / ncta * 1e-3, acc[3] / ncta * 1e-3,
          acc[4] / ncta * 1e-3, acc[5] / ncta * 1e-3, acc[6] / ncta * 1e-3);
  // per query-tile index I averages
  for (int I = 0; I < g.c / 128; ++I) {
    double a = 0, b = 0;
    size_t cnt = 0;
    for (size_t c = I; c < ncta; c += g.c / 128) {
      a += (double)(h[c * 64 + 6] - h[c * 64 + 0]);
      b += (double)(h[c * 64 + 3] - h[c * 64 + 0]);
      ++cnt;
    }
    fprintf(stderr, "   I=%d mean total %.2f us, genA %.2f us\n", I, a / cnt * 1e-3, b / cnt * 1e-3);
  }
  // detailed phase-B timeline of the I=7 CTAs (first stream/chunk with k>=1)
  for (size_t c = 7 + (size_t)(g.c / 128); c < ncta && c < 7 + 3 * (size_t)(g.c / 128); c += g.c / 128) {
    unsigned long long* r = &h[c * 64];
    fprintf(stderr, "   cta %zu (us from start): mmaA_done %.2f\n", c, (r[1] - r[0]) * 1e-3);
    for (int J = 0; J < 8; ++J)
      fprintf(stderr, "     J=%d kv_issue %.2f S_issued %.2f s_full_seen %.2f p_arrive %.2f p_seen %.2f\n", J,
              ((long long)(r[8 + J] - r[0])) * 1e-3, ((long long)(r[16 + J] - r[0])) * 1e-3,
              ((long long)(r[32 + J] - r[0])) * 1e-3, ((long long)(r[40 + J] - r[0])) * 1e-3,
              ((long long)(r[24 + J] - r[0])) * 1e-3);
  }
}

int tc_forward(const Geo& g, const void* q, const void* k, const void* v, const float* log_g, void* y, float* rowsum,
               void* ws, cudaStream_t st) {
  size_t need;
  TcFwdWs w = carve_fwd(g, ws, &need);
  const int with_den = (g.normalize || rowsum) ? 1 : 0;
  CUtensorMap m_q, m_k, m_v, m_v64, m_kt;
  if (!make_map_4d(&m_q, q, g, 128) || !make_map_4d(&m_k, k, g, 128) || !make_map_4d(&m_v, v, g, 128) ||
      !make_map_4d(&m_v64, v, g, 64) || !make_map_xt(&m_kt, w.kt, g)) {
    set_error("cuTensorMapEncodeTiled failed");
    return 3;
  }
  cudaMemsetAsync(w.zflag, 0, 4, st);
  {
    StageTimer tmr("fwd_prep", st);
    k_tc_prep_gates<<<(g.ns * g.n + 3) / 4, 128, 0, st>>>(g, log_g, w.ell, w.lamlog);
    k_tc_prep_xt<<<dim3(g.c / 64, g.n, g.ns), 256, 0, st>>>(g, (const __nv_bfloat16*)k, w.ell, w.lamlog, 0, w.kt);
  }
  {
    StageTimer tmr("fwd_update_state", st);
    cudaFuncSetAttribute(k_tc_featmajor<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, fm::SMEM);
    k_tc_featmajor<false><<<dim3((NTH + 3) / 4, g.n, g.ns), 256, fm::SMEM, st>>>(m_kt, m_v64, m_v64, g, with_den,
                                                                                 w.sp);
  }
  {
    StageTimer tmr("fwd_discumsum", st);
    k_tc_scan_fwd<<<dim3(NFB, g.ns), 256, 0, st>>>(g, with_den ? UW : 64, w.lamlog, w.sp, w.st);
  }
  {
    StageTimer tmr("fwd_attn_query", st);
    cudaFuncSetAttribute(k_tc_out, cudaFuncAttributeMaxDynamicSharedMemorySize, outk::SMEM);
    k_tc_out<<<dim3(g.c / 128, g.n, g.ns), 256, outk::SMEM, st>>>(m_q, m_k, m_v, g, (const __nv_bfloat16*)q, w.ell,
                                                                  w.st, with_den, (__nv_bfloat16*)y, rowsum, w.y32,
                                                                  w.zflag, dbg_buf(g));
  }
  dbg_report(g, st);
  count_launch(5);
  return cuda_check("tc forward");
}

// backward (interim): recompute the forward with the fp32 CUDA-core kernels
// into the backward workspace and run their backward.  The tensor-core
// backward replaces this.
size_t tc_bwd_workspace_bytes(const Geo& g) {
  return simt_fwd_bytes(g) + simt_bwd_bytes(g) + a256(4ull * g.ns * g.t) + a256(2ull * g.ns * g.t * g.e);
}

int tc_backward(const Geo& g, const void* q, const void* k, const void* v, const float* log_g, const void* y,
                const float* rowsum, const void* dy, void* dq, void* dk, void* dv, float* dlog_g, const void*,
                void* bwd_ws, cudaStream_t st) {
  const size_t f = simt_fwd_bytes(g), fb = simt_bwd_bytes(g);
  SimtWs w = simt_carve_fwd(g, bwd_ws);
  SimtBwdWs b = simt_carve_bwd(g, (char*)bwd_ws + f);
  float* r32 = (float*)((char*)bwd_ws + f + fb);
  void* yscr = (char*)r32 + a256(4ull * g.ns * g.t);
  cudaMemsetAsync(w.zflag, 0, 4, st);
  if (int rc = simt_build_table(g.p, g.d, g.D, w.idx, w.wt, st)) return rc;
  // y / rowsum recomputed into scratch (the caller's copies stay untouched)
  {
    StageTimer tmr("bwd_recompute_fp32", st);
    if (int rc = simt_forward(g, 1, q, k, v, log_g, yscr, r32, w, st)) return rc;
  }
  (void)y;
  (void)rowsum;
  StageTimer tmr("bwd_fp32", st);
  return simt_backward(g, 1, q, k, v, yscr, r32, dy, dq, dk, dv, dlog_g, w, b, st);
}

}  // namespace pa
