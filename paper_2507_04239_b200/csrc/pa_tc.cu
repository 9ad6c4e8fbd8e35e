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

#include <algorithm>
#include <utility>

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
// update_state: S'_k[block-order feature, u] = sum_j phi'(k~_j) [v_j | 1]
// grid (group of 4 tiles, chunk, stream); 128 threads
// ==========================================================================
namespace upd {
constexpr int STAGES = 4;           // 64-token TMA stages
constexpr int TOK = 64;
constexpr int KT_BYTES = 64 * 128;  // 64 dims x 64 tokens bf16
constexpr int V_BYTES = 64 * 128;   // 64 tokens x 64 values bf16
constexpr int SMEM_USED = 1024 + STAGES * (KT_BYTES + V_BYTES) + 2048 + 256;
// ask for > half the SM so one CTA (and one 512-column TMEM allocation) per SM
constexpr int SMEM = SMEM_USED > 120 * 1024 ? SMEM_USED : 120 * 1024;
}  // namespace upd

__global__ void __launch_bounds__(128, 1) k_tc_upd(const __grid_constant__ CUtensorMap tm_kt,
                                                   const __grid_constant__ CUtensorMap tm_v, Geo g, int with_den,
                                                   float* sout) {
  using namespace upd;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* kt_s = smem;
  uint8_t* v_s = smem + STAGES * KT_BYTES;
  uint8_t* ones = v_s + STAGES * V_BYTES;
  uint64_t* bars = (uint64_t*)(ones + 2048);
  uint64_t* full = bars;                // [STAGES]
  uint64_t* mdone = bars + STAGES;      // [2]
  uint64_t* fin = bars + STAGES + 2;    // [1]
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int grp = blockIdx.x, k = blockIdx.y, s = blockIdx.z;
  const int t0 = grp * 4, nt = min(4, NTH - t0);
  const int nsub = g.c / 32;   // 32-token sub-steps
  const int nstage = g.c / TOK;

  if (w == 0) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&full[i], 1);
    mbar_init(&mdone[0], 1);
    mbar_init(&mdone[1], 1);
    mbar_init(fin, 1);
    fence_barrier_init();
  }
  // ones block: K-major rows n = 0..15 of 64 tokens; row 0 all ones
  for (int i = tid; i < 2048 / 4; i += 128) ((uint32_t*)ones)[i] = (i < 32) ? 0x3F803F80u : 0u;
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  auto acc = [&](int t) { return tm + (uint32_t)(t * UW); };
  auto astage = [&](int t, int b) { return tm + 320u + (uint32_t)((t * 2 + b) * 16); };

  const int row0 = (s * g.n + k) * HD;  // K~^T rows of this chunk
  const int bi = s / g.h, hi = s % g.h;
  auto issue = [&](int j) {
    const int st = j % STAGES;
    mbar_expect_tx(&full[st], KT_BYTES + V_BYTES);
    tma_load_2d(kt_s + st * KT_BYTES, &tm_kt, &full[st], j * TOK, row0);
    tma_load_4d(v_s + st * V_BYTES, &tm_v, &full[st], 0, hi, k * g.c + j * TOK, bi);
  };
  if (tid == 0) {
    tma_prefetch(&tm_kt);
    tma_prefetch(&tm_v);
    for (int j = 0; j < min(2, nstage); ++j) issue(j);
  }

  // this thread's features in each tile: a = 4 al + l/8, b = 8 be + l%8
  int ra[4], rb[4];
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const int blk = (t0 + t) * 4 + w;
    const int bb = (t < nt) ? blk : 0;
    ra[t] = 4 * c_blk.al[bb] + (l >> 3);
    rb[t] = 8 * c_blk.be[bb] + (l & 7);
  }
  const uint32_t lane_off = (uint32_t)(w * 32) << 16;
  const uint32_t idesc64 = idesc_bf16(128, 64, false, true);
  const uint32_t idesc16 = idesc_bf16(128, 16, false, false);

  for (int i = 0; i < nsub; ++i) {
    const int j = i >> 1, h = i & 1, st = j % STAGES, buf = i & 1;
    if (i >= 2) mbar_wait(&mdone[buf], ((i - 2) >> 1) & 1);
    // stage j+2 reuses the buffer of stage j-2, whose MMAs completed (in-order) before sub-step i-2
    if (tid == 0 && h == 0 && j + 2 < nstage) issue(j + 2);
    mbar_wait(&full[st], (j / STAGES) & 1);
    const uint8_t* kts = kt_s + st * KT_BYTES;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (t < nt) {
        uint32_t va[16], vb[16], o[16];
#pragma unroll
        for (int c4 = 0; c4 < 4; ++c4) {
          const int ch = h * 4 + c4;
          *(uint4*)&va[c4 * 4] = *(const uint4*)(kts + sw128_off(ra[t], ch));
          *(uint4*)&vb[c4 * 4] = *(const uint4*)(kts + sw128_off(rb[t], ch));
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) o[c] = hmul2_bf16(va[c], vb[c]);
        tmem_st16(astage(t, buf) + lane_off, o);
      }
    }
    tc_wait_st();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint8_t* vs = v_s + st * V_BYTES;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        if (t < nt) {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const uint32_t a_t = astage(t, buf) + kk * 8;
            const uint64_t bd = smem_desc(smem_u32(vs) + (h * 32 + kk * 16) * 128, 8192, 1024, 2);
            mma_ts(acc(t), a_t, bd, idesc64, (i > 0 || kk > 0) ? 1u : 0u);
            if (with_den) {
              const uint64_t od = smem_desc(smem_u32(ones) + ((h * 2 + kk) & 3) * 32, 16, 1024, 2);
              mma_ts(acc(t) + 64, a_t, od, idesc16, (i > 0 || kk > 0) ? 1u : 0u);
            }
          }
        }
      }
      tc_commit(&mdone[buf]);
      if (i == nsub - 1) tc_commit(fin);
    }
  }
  mbar_wait(fin, 0);
  tc_fence_after();
  // epilogue: lane = feature row; write 64 (+16) fp32 columns
  const int ncols = with_den ? UW : 64;
  for (int t = 0; t < nt; ++t) {
    float* dst = sout + (((size_t)(s * g.n + k) * FH) + (size_t)(t0 + t) * 128 + w * 32 + l) * UW;
    for (int c0 = 0; c0 < ncols; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(acc(t) + lane_off + c0, r);
      tc_wait_ld();
#pragma unroll
      for (int c = 0; c < 16; c += 4)
        *(float4*)(dst + c0 + c) = make_float4(__uint_as_float(r[c]), __uint_as_float(r[c + 1]),
                                               __uint_as_float(r[c + 2]), __uint_as_float(r[c + 3]));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tm);
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
// grid (query tile of 128, chunk, stream); 128 threads
// ==========================================================================
namespace outk {
constexpr int QB = 128 * 128;           // Q tile bytes (128 tok x 64 dims bf16)
constexpr int KB = 128 * 128;           // K tile
constexpr int VB = 128 * 128;           // V tile
constexpr int STB = UW * 128;           // state block (80 u x 64 f bf16)
constexpr int KV_STAGES = 3;
constexpr int ST_STAGES = 3;
constexpr int SMEM = 1024 + QB + KV_STAGES * (KB + VB) + ST_STAGES * STB + 2048 + 4096 + 2 * 512 + 512;
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

struct OutCtx {
  uint32_t tm, lane_off;
  uint32_t* qp;  // 32 bf16x2 of q~ (registers via reference)
  uint8_t* st_s;
  uint64_t* st_full;
  uint64_t* mmaA;
  const __nv_bfloat16* st_src;  // A'_{k-1} blocks
  int tid, with_den;
};

template <int FB>
__device__ __forceinline__ void out_state_block(OutCtx& cx, uint32_t (&qp)[32]) {
  using namespace outk;
  const int bb = FB & 1;
  if (FB >= 2) mbar_wait(&cx.mmaA[bb], ((FB - 2) >> 1) & 1);
  if (cx.tid == 0 && FB + 1 < NFB) {
    const int sb = (FB + 1) % ST_STAGES;
    const uint32_t bytes = cx.with_den ? STB : 64 * 128;
    mbar_expect_tx(&cx.st_full[sb], bytes);
    bulk_load(cx.st_s + sb * STB, cx.st_src + (size_t)(FB + 1) * (UW * 64), bytes, &cx.st_full[sb]);
  }
  uint32_t o[32];
  gen_block<FB>(qp, o, std::make_integer_sequence<int, 32>{});
  const uint32_t ast = cx.tm + 128u + (uint32_t)(bb * 32);
  tmem_st16(ast + cx.lane_off, o);
  tmem_st16(ast + cx.lane_off + 16, o + 16);
  tc_wait_st();
  tc_fence_before();
  __syncthreads();
  if (cx.tid == 0) {
    tc_fence_after();
    const int sb = FB % ST_STAGES;
    mbar_wait(&cx.st_full[sb], (FB / ST_STAGES) & 1);
    const uint32_t sbase = smem_u32(cx.st_s + sb * STB);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t acc_flag = (FB > 0 || kk > 0) ? 1u : 0u;
      mma_ts(cx.tm, ast + kk * 8, smem_desc(sbase + kk * 32, 16, 1024, 2), idesc_bf16(128, 64, false, false),
             acc_flag);
      if (cx.with_den)
        mma_ts(cx.tm + 64, ast + kk * 8, smem_desc(sbase + 8192 + kk * 32, 16, 1024, 2),
               idesc_bf16(128, 16, false, false), acc_flag);
    }
    tc_commit(&cx.mmaA[bb]);
  }
  if constexpr (FB + 1 < NFB) out_state_block<FB + 1>(cx, qp);
}

__global__ void __launch_bounds__(128, 1) k_tc_out(const __grid_constant__ CUtensorMap tm_q,
                                                   const __grid_constant__ CUtensorMap tm_k,
                                                   const __grid_constant__ CUtensorMap tm_v, Geo g,
                                                   const __nv_bfloat16* __restrict__ qraw,
                                                   const float* __restrict__ ell,
                                                   const __nv_bfloat16* __restrict__ st_all, int with_den,
                                                   __nv_bfloat16* y, float* rowsum, float* y32, int* zflag) {
  using namespace outk;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* q_s = smem;
  uint8_t* k_s = q_s + QB;
  uint8_t* v_s = k_s + KV_STAGES * KB;
  uint8_t* st_s = v_s + KV_STAGES * VB;
  uint8_t* ones = st_s + ST_STAGES * STB;
  float* ell_s = (float*)(ones + 2048);       // [1024]
  float* cj = ell_s + 1024;                   // [2][128]
  uint64_t* bars = (uint64_t*)(cj + 256);
  uint64_t* q_full = bars;                    // 1
  uint64_t* kv_full = bars + 1;               // 3
  uint64_t* st_full = bars + 4;               // 3
  uint64_t* mmaA = bars + 7;                  // 2
  uint64_t* s_done = bars + 9;                // 2
  uint64_t* pv_done = bars + 11;              // 2
  uint64_t* fin = bars + 13;                  // 1
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int I = blockIdx.x, k = blockIdx.y, s = blockIdx.z;
  const int bi = s / g.h, hi = s % g.h;
  const int c0 = k * g.c;                     // chunk start token
  const int tok = c0 + I * 128 + tid;         // this thread's query token

  if (w == 0) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    for (int i = 0; i < 14; ++i) mbar_init(&bars[i], 1);
    fence_barrier_init();
  }
  for (int i = tid; i < 2048 / 4; i += 128) ((uint32_t*)ones)[i] = (i < 32) ? 0x3F803F80u : 0u;
  for (int i = tid; i < g.c; i += 128) ell_s[i] = ell[(size_t)s * g.t + c0 + i];
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  const uint32_t lane_off = (uint32_t)(w * 32) << 16;
  auto sbuf = [&](int b) { return tm + 256u + (uint32_t)(b * 128); };
  auto issue_kv = [&](int J) {
    const int st = J % KV_STAGES;
    mbar_expect_tx(&kv_full[st], KB + VB);
    tma_load_4d(k_s + st * KB, &tm_k, &kv_full[st], 0, hi, c0 + J * 128, bi);
    tma_load_4d(v_s + st * VB, &tm_v, &kv_full[st], 0, hi, c0 + J * 128, bi);
  };
  if (tid == 0) {
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_k);
    tma_prefetch(&tm_v);
    mbar_expect_tx(q_full, QB);
    tma_load_4d(q_s, &tm_q, q_full, 0, hi, c0 + I * 128, bi);
    issue_kv(0);
    if (I >= 1) issue_kv(1);
  }
  const float li = ell_s[I * 128 + tid];
  const float sig2 = g.scale * g.scale;

  // ---------------- phase A: O = phi'(q~) A'_{k-1} ----------------------
  if (k >= 1) {
    uint32_t qp[32];
    {
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
    }
    OutCtx cx{tm, lane_off, nullptr, st_s, st_full, mmaA,
              st_all + ((size_t)(s * g.n + (k - 1)) * NFB) * (UW * 64), tid, with_den};
    if (tid == 0) {
      const uint32_t bytes = with_den ? STB : 64 * 128;
      mbar_expect_tx(&st_full[0], bytes);
      bulk_load(st_s, cx.st_src, bytes, &st_full[0]);
    }
    out_state_block<0>(cx, qp);
  }

  // ---------------- phase B: intra-chunk blocks J = 0..I -----------------
  mbar_wait(q_full, 0);
  for (int J = 0; J <= I; ++J) {
    const int sb = J & 1, st = J % KV_STAGES;
    if (tid == 0) {
      tc_fence_after();
      mbar_wait(&kv_full[st], (J / KV_STAGES) & 1);
      if (J >= 2) mbar_wait(&pv_done[sb], ((J - 2) >> 1) & 1);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        mma_ss(sbuf(sb), smem_desc(smem_u32(q_s) + kk * 32, 16, 1024, 2),
               smem_desc(smem_u32(k_s + st * KB) + kk * 32, 16, 1024, 2), idesc_bf16(128, 128, false, false),
               kk > 0 ? 1u : 0u);
      tc_commit(&s_done[sb]);
    }
    // key-side decay factors for this block
    const bool diag = (J == I);
    const float lref = ell_s[J * 128 + 127];
    cj[sb * 128 + tid] = diag ? ell_s[J * 128 + tid] : __expf(lref - ell_s[J * 128 + tid]);
    __syncthreads();
    mbar_wait(&s_done[sb], (J >> 1) & 1);
    tc_fence_after();
    const float ri = diag ? 0.f : __expf(li - lref) * sig2;
#pragma unroll
    for (int ch = 0; ch < 4; ++ch) {
      uint32_t r[32], pk[16];
      tmem_ld32(sbuf(sb) + lane_off + ch * 32, r);
      tc_wait_ld();
#pragma unroll
      for (int e2 = 0; e2 < 16; ++e2) {
        float pv[2];
#pragma unroll
        for (int z = 0; z < 2; ++z) {
          const int jj = ch * 32 + e2 * 2 + z;
          const float sv = __uint_as_float(r[e2 * 2 + z]);
          if (diag)
            pv[z] = (jj <= tid) ? __expf(li - cj[sb * 128 + jj]) * sig2 * sv * sv : 0.f;
          else
            pv[z] = ri * cj[sb * 128 + jj] * sv * sv;
        }
        pk[e2] = pack_bf16(pv[0], pv[1]);
      }
      tmem_st16(sbuf(sb) + lane_off + ch * 16, pk);
    }
    tc_wait_st();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint32_t vb = smem_u32(v_s + st * VB);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t acc_flag = (k >= 1 || J > 0 || kk > 0) ? 1u : 0u;
        mma_ts(tm, sbuf(sb) + kk * 8, smem_desc(vb + kk * 2048, 8192, 1024, 2), idesc_bf16(128, 64, false, true),
               acc_flag);
        if (with_den)
          mma_ts(tm + 64, sbuf(sb) + kk * 8, smem_desc(smem_u32(ones) + (kk & 3) * 32, 16, 1024, 2),
                 idesc_bf16(128, 16, false, false), acc_flag);
      }
      tc_commit(&pv_done[sb]);
      if (J + 2 <= I) {
        if (J >= 1) mbar_wait(&pv_done[(J - 1) & 1], ((J - 1) >> 1) & 1);
        issue_kv(J + 2);
      }
      if (J == I) tc_commit(fin);
    }
  }
  mbar_wait(fin, 0);
  tc_fence_after();
  // ---------------- epilogue -------------------------------------------
  uint32_t o[64];
  tmem_ld32(tm + lane_off, o);
  tmem_ld32(tm + lane_off + 32, o + 32);
  float den = 0.f;
  if (with_den) {
    uint32_t r[16];
    tmem_ld16(tm + lane_off + 64, r);
    tc_wait_ld();
    den = __uint_as_float(r[0]);
  }
  tc_wait_ld();
  const size_t row = rowid(g, s, tok);
  float inv = 1.f;
  if (g.normalize) {
    if (!(den > 0.f)) atomicAdd(zflag, 1);
    inv = 1.f / den;
  }
  if (rowsum) rowsum[row] = den;
  uint4* yrow = (uint4*)(y + row * HD);
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
  tc_fence_before();
  __syncthreads();
  if (w == 0) tmem_dealloc<512>(tm);
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

static bool make_map_4d(CUtensorMap* m, const void* ptr, const Geo& g, int box_tokens) {
  // [b][t][h][64] bf16: dims inner -> outer {64, h, t, b}
  cuuint64_t dims[4] = {(cuuint64_t)HD, (cuuint64_t)g.h, (cuuint64_t)g.t, (cuuint64_t)g.b};
  cuuint64_t strides[3] = {(cuuint64_t)HD * 2, (cuuint64_t)g.h * HD * 2, (cuuint64_t)g.t * g.h * HD * 2};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)box_tokens, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(ptr), dims, strides, box,
                                es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static bool make_map_xt(CUtensorMap* m, const void* ptr, const Geo& g) {
  // [ns*n*64 rows][c tokens] bf16, box 64 tokens x 64 rows
  cuuint64_t dims[2] = {(cuuint64_t)g.c, (cuuint64_t)g.ns * g.n * HD};
  cuuint64_t strides[1] = {(cuuint64_t)g.c * 2};
  cuuint32_t box[2] = {64, 64};
  cuuint32_t es[2] = {1, 1};
  return cuTensorMapEncodeTiled(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                                es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
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
  k_tc_prep_gates<<<(g.ns * g.n + 3) / 4, 128, 0, st>>>(g, log_g, w.ell, w.lamlog);
  k_tc_prep_xt<<<dim3(g.c / 64, g.n, g.ns), 256, 0, st>>>(g, (const __nv_bfloat16*)k, w.ell, w.lamlog, 0, w.kt);
  cudaFuncSetAttribute(k_tc_upd, cudaFuncAttributeMaxDynamicSharedMemorySize, upd::SMEM);
  k_tc_upd<<<dim3((NTH + 3) / 4, g.n, g.ns), 128, upd::SMEM, st>>>(m_kt, m_v64, g, with_den, w.sp);
  k_tc_scan_fwd<<<dim3(NFB, g.ns), 256, 0, st>>>(g, with_den ? UW : 64, w.lamlog, w.sp, w.st);
  cudaFuncSetAttribute(k_tc_out, cudaFuncAttributeMaxDynamicSharedMemorySize, outk::SMEM);
  k_tc_out<<<dim3(g.c / 128, g.n, g.ns), 128, outk::SMEM, st>>>(m_q, m_k, m_v, g, (const __nv_bfloat16*)q, w.ell,
                                                                w.st, with_den, (__nv_bfloat16*)y, rowsum, w.y32,
                                                                w.zflag);
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
  if (int rc = simt_forward(g, 1, q, k, v, log_g, yscr, r32, w, st)) return rc;
  (void)y;
  (void)rowsum;
  return simt_backward(g, 1, q, k, v, yscr, r32, dy, dq, dk, dv, dlog_g, w, b, st);
}

}  // namespace pa
