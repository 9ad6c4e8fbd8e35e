// Forward output kernel: intra-chunk power attention + state query + combine
// + normalize (reference attention.py:273-309 per chunk, kernels.py:86-110,
// chunked.py:372-395), bf16/fp16 tcgen05 path, p = 2, d = e = 64.
//
//   y_m = O_intra_m + sigma^2 gp_m phi'(q_m) . slot_k      (O_state)
//   O_intra = sum_J P_J V_J,  P = causal pairwise-decayed (sigma q.k)^2
//
// B200 design.  One CTA per 128-query tile of a chunk, 14 warps:
//   w0..w3   generate phi'(q) (runtime block loop, x from thread-private shared
//            memory) for the state query, then run the epilogue;
//   w4..w7   turn S = Q K_J^T into P (decay, square, mask) in TMEM;
//   w8       TMEM owner;  w9 TMA for Q / K / V;  w10 bulk copies of the state;
//   w11, w12 tcgen05.mma issuers of the state query (even / odd 128-slot steps);
//   w13      tcgen05.mma issuer of the intra-chunk S and P V.
// The state query and the intra-chunk attention accumulate into separate TMEM
// accumulators (O_state, O_intra) and proceed concurrently; the epilogue
// combines them.  Each barrier wait costs ~160 cycles even when the phase is
// complete and one thread issues at most one MMA per ~45 cycles
// (profiles/README.md), so the three issuers hide each other's latencies.
#include <cuda.h>

#include "pa_common.cuh"
#include "pa_sm100.cuh"
#include "pa_tc.cuh"
#include "pa_tc_common.cuh"

namespace pa {
using namespace sm100;
using namespace tc;

static __constant__ BlkTab c_blk_o = make_blk_tab();

#ifdef PA_TRACE
// debug build only (tools/trace_out.py): clock64 stamps of one CTA
__device__ long long g_trace4[512];
extern "C" int pa_debug_trace4(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trace4, sizeof(long long) * n);
}
#define PA_TR4(c, i) \
  if (c) g_trace4[(i)] = clock64()
#else
#define PA_TR4(c, i)
#endif

struct of2 {
  float x, y;
};
__device__ __forceinline__ of2 omul2(of2 a, of2 b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(*(uint64_t*)&a), "l"(*(uint64_t*)&b));
  return *(of2*)&r;
}

namespace out2 {
constexpr int QB = 128 * 128;           // Q tile bytes (128 tok x 64 dims bf16)
constexpr int KB = 128 * 128;           // K tile
constexpr int VB = 128 * 128;           // V tile
constexpr int STB = 128 * 128;          // state step: 128 slots x 64 values
constexpr int STD = 128 * 32;           // state step score-sum part
constexpr int NSTEP = NKB / 2;          // 18 steps of 128 slots
constexpr int KV_ST = 3;
constexpr int ST_ST = 4;
constexpr int XH = 8 * 128 * 16;        // fp16 q rows, thread-private uint4 columns
constexpr int SMEM = 1024 + QB + KV_ST * (KB + VB) + ST_ST * (STB + STD) + XH + 2048 + 4096 + 1024 + 512;
constexpr int THREADS = 576;
// w0..w3 phi'(q) + epilogue, w4..w11 P (two warps per lane quadrant, 64 columns
// each), then the issuing warps on the highest ids
constexpr int W_TMEM = 12, W_TMA_KV = 13, W_TMA_ST = 14, W_MMA_ST = 15, W_MMA_IN = 17;
}  // namespace out2

template <int kDen>
__global__ void __launch_bounds__(out2::THREADS, 1) k_tc_out2(
    const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
    const __grid_constant__ CUtensorMap tm_v, Geo g, const __nv_bfloat16* __restrict__ qraw,
    const float* __restrict__ ell, const __half* __restrict__ st_main, const __half* __restrict__ st_den,
    __nv_bfloat16* y, float* rowsum, float* y32, int* zflag) {
  using namespace out2;
  constexpr bool den = kDen != 0;
  // TMEM columns: O_state [0, OW), O_intra [OW, 2 OW), phi' buffers 2 x 64, S/P buffers NSB x 128
  constexpr uint32_t OW = den ? 80u : 64u;
  constexpr uint32_t TOS = 0, TOI = OW, TA = 2 * OW;
  constexpr uint32_t TSP = TA + 128;
  constexpr int NSB = den ? 1 : 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* q_s = smem;
  uint8_t* k_s = q_s + QB;
  uint8_t* v_s = k_s + KV_ST * KB;
  uint8_t* st_s = v_s + KV_ST * VB;
  uint8_t* sd_s = st_s + ST_ST * STB;
  uint4* xh_s = (uint4*)(sd_s + ST_ST * STD);
  uint8_t* ones = (uint8_t*)(xh_s + 8 * 128);
  float* ell_s = (float*)(ones + 2048);       // [1024]
  float* cj = ell_s + 1024;                   // [2][128] column factors of the current key block
  uint64_t* bars = (uint64_t*)(cj + 256);
  uint64_t* q_full = bars;                    // 1
  uint64_t* kv_full = q_full + 1;             // KV_ST
  uint64_t* kv_empty = kv_full + KV_ST;       // KV_ST
  uint64_t* st_full = kv_empty + KV_ST;       // ST_ST
  uint64_t* st_empty = st_full + ST_ST;       // ST_ST
  uint64_t* a_full = st_empty + ST_ST;        // 2
  uint64_t* a_empty = a_full + 2;             // 2
  uint64_t* s_full = a_empty + 2;             // 2
  uint64_t* p_full = s_full + 2;              // 2
  uint64_t* pv_done = p_full + 2;             // 2
  uint64_t* a_done = pv_done + 2;             // 1 (both state issuers)
  uint64_t* fin = a_done + 1;                 // 1 (intra issuer)
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int I = blockIdx.x, k = blockIdx.y, s = blockIdx.z;
  const int bi = s / g.h, hi = s % g.h;
  const int c0 = k * g.c;
  const bool has_state = k >= 1 || g.prefix;   // state before chunk k = slot k
#ifdef PA_TRACE
  const bool trb = blockIdx.x == 7 && blockIdx.y == 5 && blockIdx.z == 3;
#else
  const bool trb = false;
#endif

  if (w == W_TMEM) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < KV_ST; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < ST_ST; ++i) {
      mbar_init(&st_full[i], 1);
      mbar_init(&st_empty[i], 2);   // a step pair: one commit per state-query issuer
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&a_full[i], 4);
      mbar_init(&a_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 8);
      mbar_init(&pv_done[i], 1);
    }
    mbar_init(a_done, 2);
    mbar_init(fin, 1);
    fence_barrier_init();
  }
  for (int i = tid; i < 2048 / 4; i += THREADS) ((uint32_t*)ones)[i] = (i < 32) ? 0x3F803F80u : 0u;
  for (int i = tid; i < g.c; i += THREADS) ell_s[i] = ell[(size_t)s * g.t + c0 + i];
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;

  if (w == W_TMA_KV) {
    // one issuing lane per tensor: a thread completes one TMA copy per ~610 cycles
    // whatever its size (profiles/r01_bulk_copy_probe.txt)
    if (l < 2) {
      if (l == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        mbar_expect_tx(q_full, QB);
        tma_load_4d(q_s, &tm_q, q_full, 0, hi, c0 + I * 128, bi);
      }
      for (int J = 0; J <= I; ++J) {
        const int st = J % KV_ST;
        if (J >= KV_ST) mbar_wait(&kv_empty[st], ((J / KV_ST) + 1) & 1);
        if (l == 0) mbar_expect_tx(&kv_full[st], KB + VB);
        __syncwarp(3u);
        if (l == 0) tma_load_4d(k_s + st * KB, &tm_k, &kv_full[st], 0, hi, c0 + J * 128, bi);
        if (l == 1) tma_load_4d(v_s + st * VB, &tm_v, &kv_full[st], 0, hi, c0 + J * 128, bi);
      }
    }
  } else if (w == W_TMA_ST) {
    constexpr int NL = den ? 3 : 2;
    if (l < NL && has_state) {
      const __half* srcm = st_main + (size_t)(s * g.nsl + k) * ((size_t)FH * 64);
      const __half* srcd = st_den + (size_t)(s * g.nsl + k) * ((size_t)FH * 16);
      // a PAIR of 128-slot steps per barrier, one 16 KB copy per lane: a thread
      // completes one copy per ~690 cycles whatever its size
      // (profiles/r01_bulk_copy_probe.txt), lanes overlap
      for (int stp = 0; stp < NSTEP; stp += 2) {
        const int sb = stp % ST_ST;   // 0 or 2: the pair occupies slots sb, sb + 1
        if (stp >= ST_ST) mbar_wait(&st_empty[sb], ((stp / ST_ST) + 1) & 1);
        if (l == 0) mbar_expect_tx(&st_full[sb], 2 * (STB + (den ? STD : 0)));
        __syncwarp((1u << NL) - 1u);
        if (l < 2) bulk_load(st_s + (sb + l) * STB, srcm + (size_t)(stp + l) * 128 * 64, STB, &st_full[sb]);
        if (den && l == 2) bulk_load(sd_s + sb * STD, srcd + (size_t)stp * 128 * 16, 2 * STD, &st_full[sb]);
      }
    }
  } else if (w == W_MMA_ST || w == W_MMA_ST + 1) {
    // ---------------- state query: O_state += phi'(q) slot_k ------------------
    {
      const int mw = w - W_MMA_ST;
      if (has_state) {
        constexpr uint32_t id64mn_h = idesc_f16(128, 64, false, true);
        constexpr uint32_t id16mn_h = idesc_f16(128, 16, false, true);
        const uint64_t sm0 = smem_desc(smem_u32(st_s), 8192, 1024, 2);
        const uint64_t sd0 = smem_desc(smem_u32(sd_s), 2048, 256, 6);
        PA_TR4(trb && mw == 0, 0);
        // deterministic mode: w15 issues every step in order (one summation order)
        const int sstep = g.det ? 1 : 2;
        for (int stp = g.det ? (mw ? NSTEP : 0) : mw; stp < NSTEP; stp += sstep) {
          const int bb = stp & 1, sb = stp % ST_ST;
          mbar_wait_w(&a_full[bb], (stp >> 1) & 1);
          PA_TR4(trb, 10 + stp * 3 + 0);
          mbar_wait_w(&st_full[sb & ~1], (stp / ST_ST) & 1);
          PA_TR4(trb, 10 + stp * 3 + 1);
          tc_fence_after();
          const uint64_t so = (uint64_t)((sb * STB) >> 4), sdo = (uint64_t)((sb * STD) >> 4);
          const uint32_t ab = tm + TA + (uint32_t)(bb * 64);
          // both issuers accumulate into the zero-initialised O_state
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {   // 16 slots per MMA: 2048 B of [slot][64] rows, 512 B of [slot][16]
            mma_ts_w(tm + TOS, ab + kk * 8, sm0 + so + (uint64_t)(kk * 128), id64mn_h, 1u);
            if (den) mma_ts_w(tm + TOS + 64, ab + kk * 8, sd0 + sdo + (uint64_t)(kk * 32), id16mn_h, 1u);
          }
          tc_commit_w(&a_empty[bb]);
          tc_commit_w(&st_empty[sb & ~1]);
          PA_TR4(trb, 10 + stp * 3 + 2);
        }
      }
      tc_commit_w(a_done);
    }
  } else if (w == W_MMA_IN) {
    // ---------------- intra-chunk: S = Q K_J^T, O_intra += P V_J ---------------
    {
      constexpr uint32_t id128 = idesc_bf16(128, 128, false, false);
      constexpr uint32_t id64mn = idesc_bf16(128, 64, false, true);
      constexpr uint32_t id16k = idesc_bf16(128, 16, false, false);
      const uint64_t qd0 = smem_desc(smem_u32(q_s), 16, 1024, 2);
      const uint64_t kd0 = smem_desc(smem_u32(k_s), 16, 1024, 2);
      const uint64_t vd0 = smem_desc(smem_u32(v_s), 8192, 1024, 2);
      const uint64_t od0 = smem_desc(smem_u32(ones), 16, 1024, 2);
      mbar_wait_w(q_full, 0);
      auto issue_s = [&](int J) {
        const int st = J % KV_ST, sb = J % NSB;
        mbar_wait_w(&kv_full[st], (J / KV_ST) & 1);
        if (J >= NSB) mbar_wait_w(&pv_done[sb], ((J / NSB) + 1) & 1);
        tc_fence_after();
        const uint64_t ko = (uint64_t)((st * KB) >> 4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ss_w(tm + TSP + (uint32_t)(sb * 128), qd0 + (uint64_t)(kk * 2), kd0 + ko + (uint64_t)(kk * 2), id128,
                 kk > 0 ? 1u : 0u);
        tc_commit_w(&s_full[sb]);
      };
      issue_s(0);
      for (int J = 0; J <= I; ++J) {
        if (NSB == 2 && J + 1 <= I) issue_s(J + 1);
        const int sb = J % NSB, st = J % KV_ST;
        PA_TR4(trb, 100 + J * 3 + 0);
        mbar_wait_w(&p_full[sb], (J / NSB) & 1);
        PA_TR4(trb, 100 + J * 3 + 1);
        tc_fence_after();
        const uint64_t vo = (uint64_t)((st * VB) >> 4);
        const uint32_t pb = tm + TSP + (uint32_t)(sb * 128);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t f = (J > 0 || kk > 0) ? 1u : 0u;
          mma_ts_w(tm + TOI, pb + kk * 8, vd0 + vo + (uint64_t)(kk * 128), id64mn, f);
          if (den) mma_ts_w(tm + TOI + 64, pb + kk * 8, od0 + (uint64_t)((kk & 3) * 2), id16k, f);
        }
        tc_commit_w(&pv_done[sb]);
        tc_commit_w(&kv_empty[st]);
        PA_TR4(trb, 100 + J * 3 + 2);
        if (NSB == 1 && J + 1 <= I) issue_s(J + 1);
      }
      tc_commit_w(fin);
    }
  } else if (w < 4) {
    // ---------------- phi'(q) generation, then the epilogue --------------------
    const int q = w, row = q * 32 + l;          // TMEM lane == query row in the tile
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int tok = c0 + I * 128 + row;
    const float li = ell_s[I * 128 + row];
    const float sig2 = g.scale * g.scale;
    if (has_state) {
      {
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
        for (int c = 0; c < (int)OW; c += 16) tmem_st16(tm + TOS + lane_off + c, z);
        // phi'(q) from the exact bf16 q (one rounding per feature); the query
        // scale sigma^2 gp_m (chunked.py:379-385) multiplies the fp32 result
        const uint4* src = (const uint4*)(qraw + rowid(g, s, tok) * HD);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          const uint4 v4 = src[c8];
          const uint32_t* pv = (const uint32_t*)&v4;
          uint4 h4;
          uint32_t* ph = (uint32_t*)&h4;
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            const float2 f2 = __bfloat1622float2(*(const __nv_bfloat162*)&pv[e2]);
            ph[e2] = pack_f16(f2.x, f2.y);
          }
          xh_s[c8 * 128 + row] = h4;
        }
      }
#pragma unroll 1
      for (int stp = 0; stp < NSTEP; ++stp) {
        const int bb = stp & 1;
        PA_TR4(trb && w == 0 && l == 0, 200 + stp * 2 + 0);
        if (stp >= 2) mbar_wait(&a_empty[bb], ((stp >> 1) + 1) & 1);
        PA_TR4(trb && w == 0 && l == 0, 200 + stp * 2 + 1);
        const uint32_t ab = tm + TA + (uint32_t)(bb * 64) + lane_off;
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const int blk = stp * 4 + f, al = c_blk_o.al[blk], be = c_blk_o.be[blk];
          const uint2 xa = *(const uint2*)((const uint32_t*)&xh_s[(al >> 1) * 128 + row] + (al & 1) * 2);
          const uint4 xb = xh_s[be * 128 + row];
          const uint32_t xbv[4] = {xb.x, xb.y, xb.z, xb.w};
          const uint32_t bc[4] = {__byte_perm(xa.x, 0, 0x1010), __byte_perm(xa.x, 0, 0x3232),
                                  __byte_perm(xa.y, 0, 0x1010), __byte_perm(xa.y, 0, 0x3232)};
          uint32_t o[16];
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int jp = 0; jp < 4; ++jp) o[i * 4 + jp] = hmul2_f16(bc[i], xbv[jp]);
          tmem_st16(ab + (uint32_t)(f * 16), o);
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (l == 0) mbar_arrive(&a_full[bb]);
      }
    }
    // ---------------- epilogue: y = cm O_state + O_intra -------------------------
    PA_TR4(trb && w == 0 && l == 0, 300);
    if (has_state) mbar_wait(a_done, 0);
    PA_TR4(trb && w == 0 && l == 0, 301);
    mbar_wait(fin, 0);
    PA_TR4(trb && w == 0 && l == 0, 302);
    tc_fence_after();
    const float cm = has_state ? sig2 * __expf(li) / pow2_neg_bits(g.k0 + k - 1) : 0.f;  // undo the slot scale
    uint32_t oi[64];
    tmem_ld32(tm + TOI + lane_off, oi);
    tmem_ld32(tm + TOI + lane_off + 32, oi + 32);
    float yv[64];
    tc_wait_ld();
#pragma unroll
    for (int i = 0; i < 64; ++i) yv[i] = __uint_as_float(oi[i]);
    if (has_state) {
      tmem_ld32(tm + TOS + lane_off, oi);
      tmem_ld32(tm + TOS + lane_off + 32, oi + 32);
      tc_wait_ld();
#pragma unroll
      for (int i = 0; i < 64; ++i) yv[i] = fmaf(cm, __uint_as_float(oi[i]), yv[i]);
    }
    float dn = 0.f;
    if (den) {
      uint32_t r[16];
      tmem_ld16(tm + TOI + 64 + lane_off, r);
      tc_wait_ld();
      dn = __uint_as_float(r[0]);
      if (has_state) {
        tmem_ld16(tm + TOS + 64 + lane_off, r);
        tc_wait_ld();
        dn = fmaf(cm, __uint_as_float(r[0]), dn);
      }
    }
    const size_t rw = rowid(g, s, tok);
    float inv = 1.f;
    if (g.normalize) {
      if (tok >= g.treal) {
        inv = 0.f;   // zero padding past the sequence end (partial last chunk): y = 0
      } else {
        if (!(dn > 0.f)) atomicAdd(zflag, 1);
        inv = 1.f / dn;
      }
    }
    if (rowsum) rowsum[rw] = dn;
    {
      // y rows go out through shared memory (the drained state stages; 32 rows x
      // 144 B per warp, padded against bank conflicts): each warp store writes four
      // whole 128-byte rows instead of 32 scattered 16-byte pieces
      uint8_t* stg = st_s + w * (32 * 144);
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8)
        *(uint4*)(stg + l * 144 + c8 * 16) =
            make_uint4(pack_bf16(yv[c8 * 8] * inv, yv[c8 * 8 + 1] * inv),
                       pack_bf16(yv[c8 * 8 + 2] * inv, yv[c8 * 8 + 3] * inv),
                       pack_bf16(yv[c8 * 8 + 4] * inv, yv[c8 * 8 + 5] * inv),
                       pack_bf16(yv[c8 * 8 + 6] * inv, yv[c8 * 8 + 7] * inv));
      __syncwarp();
#pragma unroll
      for (int r4 = 0; r4 < 32; r4 += 4) {
        const int rw4 = r4 + (l >> 3), c8 = l & 7;
        *(uint4*)(y + rowid(g, s, tok - l + rw4) * HD + c8 * 8) = *(const uint4*)(stg + rw4 * 144 + c8 * 16);
      }
    }
    if (g.normalize && y32) {
      // fp32 y rows (read by the backward prologue): the warp's 32 rows are one
      // contiguous 8 KB block of the stream-major buffer -- staged (32 x 68 floats,
      // after the bf16 rows above) and stored as consecutive 16-byte runs
      __syncwarp();
      float* sf = (float*)(st_s + 4 * (32 * 144)) + w * (32 * 68);
#pragma unroll
      for (int c4 = 0; c4 < 16; ++c4)
        *(float4*)(sf + l * 68 + c4 * 4) =
            make_float4(yv[c4 * 4] * inv, yv[c4 * 4 + 1] * inv, yv[c4 * 4 + 2] * inv, yv[c4 * 4 + 3] * inv);
      __syncwarp();
      float* dst0 = y32 + ((size_t)s * g.t + tok - l) * HD;
#pragma unroll 4
      for (int i = l; i < 32 * 16; i += 32) {
        const int rw = i >> 4, cc = i & 15;
        *(float4*)(dst0 + (size_t)rw * HD + cc * 4) = *(const float4*)(sf + rw * 68 + cc * 4);
      }
    }
  } else if (w < 12) {
    // ---------------- P = decayed (sigma q.k)^2 under the causal mask ------------
    // two warps per lane quadrant: half ph takes S columns [64 ph, 64 ph + 64)
    const int q = w & 3, row = q * 32 + l, ph = (w - 4) >> 2;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const float li = ell_s[I * 128 + row];
    const float sig2 = g.scale * g.scale;
    for (int J = 0; J <= I; ++J) {
      const int sb = J % NSB, cb = J & 1;
      const bool diag = (J == I);
      const float lref = ell_s[J * 128 + 127];
      if (ph == 0) cj[cb * 128 + row] = diag ? ell_s[J * 128 + row] : __expf(lref - ell_s[J * 128 + row]);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      PA_TR4(trb && w == 4 && l == 0, 400 + J * 3 + 0);
      mbar_wait(&s_full[sb], (J / NSB) & 1);
      PA_TR4(trb && w == 4 && l == 0, 400 + J * 3 + 1);
      tc_fence_after();
      const float ri = __expf(li - lref) * sig2;
      const float* cjs = cj + cb * 128;
      const uint32_t sp = tm + TSP + (uint32_t)(sb * 128) + lane_off;
      uint32_t rb[2][32];
      tmem_ld32(sp + ph * 64, rb[0]);
      tmem_ld32(sp + ph * 64 + 32, rb[1]);
      tc_wait_ld();
      // P is written back in place as bf16 pairs: the half-1 warp's P lands on S
      // columns [32, 64), which the half-0 warp of this quadrant must have read
      asm volatile("bar.sync %0, 64;" ::"r"(2 + q) : "memory");
#pragma unroll
      for (int ch = 2 * ph; ch < 2 * ph + 2; ++ch) {
        uint32_t pk[16];
        const uint32_t* r = rb[ch & 1];
        if (!diag) {
          // P = r_i c_j s^2 in packed f32x2 arithmetic (3 FMUL2 per pair)
          const of2 ri2 = {ri, ri};
#pragma unroll
          for (int e4 = 0; e4 < 8; ++e4) {
            const float4 c4 = *(const float4*)(cjs + ch * 32 + e4 * 4);
#pragma unroll
            for (int z = 0; z < 2; ++z) {
              const of2 sv = {__uint_as_float(r[e4 * 4 + 2 * z]), __uint_as_float(r[e4 * 4 + 2 * z + 1])};
              const of2 cc = z ? of2{c4.z, c4.w} : of2{c4.x, c4.y};
              const of2 pv = omul2(omul2(omul2(sv, sv), cc), ri2);
              pk[e4 * 2 + z] = pack_bf16(pv.x, pv.y);
            }
          }
        } else {
          // diagonal block: exact pairwise decay exp(ell_i - ell_j), causal mask j <= i
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
        }
        tmem_st16(sp + ch * 16, pk);
      }
      tc_wait_st();
      PA_TR4(trb && w == 4 && l == 0, 400 + J * 3 + 2);
      tc_fence_before();
      __syncwarp();
      if (l == 0) mbar_arrive(&p_full[sb]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == W_TMEM) tmem_dealloc<512>(tm);
}

int tc_out(const Geo& g, const CUtensorMap& m_q, const CUtensorMap& m_k, const CUtensorMap& m_v, const void* q,
           const float* ell, const __half* st_main, const __half* st_den, int with_den, void* y, float* rowsum,
           float* y32, int* zflag, cudaStream_t st) {
  using namespace out2;
  auto fn = with_den ? k_tc_out2<1> : k_tc_out2<0>;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  fn<<<dim3(g.c / 128, g.n, g.ns), THREADS, SMEM, st>>>(m_q, m_k, m_v, g, (const __nv_bfloat16*)q, ell, st_main,
                                                        st_den, (__nv_bfloat16*)y, rowsum, y32, zflag);
  return 0;
}

}  // namespace pa
