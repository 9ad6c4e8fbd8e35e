// State VJP as one tensor-core GEMM per gradient (reference gradients.py:46-76
// expand_vjp, 191-213 update-state VJP, 406-431 query-state VJP), bf16/fp16
// tcgen05 path, p = 2, d = e = 64.
//
// For phi'(x)_ab = x_a x_b the state VJP of a token with row vector u
// (u = dnum on the query side, [v | 1] on the update side) is
//     dx_c = sum_b x_b sum_e u_e T_{cb,e}
// with T the state expanded to all 64 x 64 ordered pairs (T_{cb} = slot(min,max),
// doubled on the diagonal: the omega weight of the stored slots makes this the
// exact derivative).  So dx = Z E with Z_m = x_m (x) u_m (4096 products per
// token) and E the expanded state as a [64 c] x [64 b * 64 e] matrix: one
// M = 128 tokens, N = 64, K = 4096 GEMM with the A operand generated into TMEM
// (one HMUL2 per two products, no loads) and E streamed as 64 tiles of
// [64 c][64 e] (8 KB, SW128, written by the backward scan).  The earlier
// formulation (dphi = u S^T on the tensor core, then the expand-VJP on the FMA
// pipe) read every dphi value back from TMEM and was bound by that (~64 B/clk).
//
//   query  (kUpd = false): dq_m = sigma^2 gp_m (Z E(A'_{k-1}))_m      256 tokens per CTA
//                          dell_m += <dq~, q~>/2
//   update (kUpd = true):  dk_j = W_j (Z E(dS~_k))_j, cu_j = <dk~, k~>/2   128 tokens per CTA
//                          dv_j = W_j/2 (Y E(dS~_k))_j with Y_j = k_j (x) k_j over
//                          the same tile used MN-major (K = c, N = e): the sum over
//                          ordered pairs counts every unordered pair twice.
// Score sum (normalize): one more tile E_G[c][b] (the key-sum column) with
// A = x * dden (query) or A = x (update, dk only).
//
// Persistent, one CTA per SM, tiles of (stream, chunk, token block) strided over
// the grid.  Warp roles: w0..w7 generate A (group gq = w/4 owns TMEM lane
// quadrant w%4; query: gq = token half, update: gq = 0 -> Z (dk), 1 -> Y (dv));
// w8 TMA (E tiles); w9/w10 MMA issuers over alternating stages; w11..w18
// epilogue, which also prepares the scaled operand words of the tile after next
// (double-buffered in shared memory, so the generators never wait on HBM).  TMEM: one accumulator [0, 128), zeroed and handed back by
// the epilogue right after it is read (the stores run under the next tile's
// MMAs, the generators run up to three stages into the next tile); A stages
// 3 x 128 columns [128, 512) (two E tiles x two groups x 32 columns): 16 MMAs
// per stage amortise the issuers' barrier round trips (~160 cycles per wait even
// on a completed phase).  Measured limit (tools/trace_zv.py): the generate ->
// MMA -> release round trip (~1400 cycles) over three stages, so the two
// issuers rarely overlap and run at the single-issuer rate (tools/ts_contention.cu:
// 44 cycles per N = 64 MMA with eight warps storing to TMEM; two issuers 32).
#include <cuda.h>

#include "pa_common.cuh"
#include "pa_sm100.cuh"
#include "pa_tc.cuh"
#include "pa_tc_common.cuh"

namespace pa {
using namespace sm100;
using namespace tc;

#ifdef PA_TRACE
// debug build only (tools/trace_zv.py): clock64 stamps of one CTA
__device__ long long g_trace6[2048];
extern "C" int pa_debug_trace6(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trace6, sizeof(long long) * n);
}
#define PA_TR6(c, i) \
  if (c) g_trace6[(i) + (kUpd ? 0 : 1024)] = clock64()
#else
#define PA_TR6(c, i)
#endif

namespace zv {
constexpr int TILE = 64 * 128;   // bytes of one E tile: 64 rows (c) x 64 fp16 (e), SW128
constexpr int NSB = 3;           // B ring: 4 E tiles (32 KB, one bulk copy) per stage
constexpr int TPS = 4;           // E tiles per B stage
constexpr int NSA = 3;           // A stages in TMEM (two E tiles each)
constexpr int NGEN = 256;        // generating threads (one token row each)
constexpr int NGW = 8;           // generating warps: 2 groups x 4 lane quadrants
constexpr int THREADS = 608;
constexpr int W_TMA = 8, W_MMA = 9, W_EPI = 11;   // MMA issuers: w9 (even stages), w10 (odd stages)
constexpr int XW = 32 * NGEN * 4;   // fp16 words of one operand for one tile, [word][thread]
// no static shared memory: the dynamic window starts 1024-aligned, so only a
// small slack is reserved (checked at run time) -- the budget is at the 227 KB limit
constexpr int SMEM_PAD = 128;
constexpr int SMEM = SMEM_PAD + NSB * TPS * TILE + 4 * XW + 2 * NGEN * 4 + 256;
}  // namespace zv

// 2^-floor(log2(m)) for m > 0 (so m * p in [1, 2)), 1 for m == 0
__device__ __forceinline__ float pow2_norm(float m) {
  if (!(m > 0.f)) return 1.f;
  const int e = ((__float_as_int(m) >> 23) & 255) - 127;
  return __int_as_float((127 - e) << 23);
}

// 8 bf16 / fp16 values: running max |x|; fp16x2 words scaled by p (a power of two)
__device__ __forceinline__ float chunk_max(uint4 v4, bool is_bf16, float m) {
  const uint32_t* pv4 = (const uint32_t*)&v4;
#pragma unroll
  for (int e2 = 0; e2 < 4; ++e2) {
    const float2 f2 = is_bf16 ? __bfloat1622float2(*(const __nv_bfloat162*)&pv4[e2])
                              : __half22float2(*(const __half2*)&pv4[e2]);
    m = fmaxf(m, fmaxf(fabsf(f2.x), fabsf(f2.y)));
  }
  return m;
}
__device__ __forceinline__ void chunk_f16(uint4 v4, bool is_bf16, float p, uint32_t* o) {
  const uint32_t* pv4 = (const uint32_t*)&v4;
#pragma unroll
  for (int e2 = 0; e2 < 4; ++e2) {
    const float2 f2 = is_bf16 ? __bfloat1622float2(*(const __nv_bfloat162*)&pv4[e2])
                              : __half22float2(*(const __half2*)&pv4[e2]);
    o[e2] = pack_f16(f2.x * p, f2.y * p);
  }
}

struct ZvTile {
  int I, k, s;
};
__device__ __forceinline__ ZvTile zv_tile(int ti, int nI, int nk, int kbeg) {
  ZvTile t;
  t.I = ti % nI;
  const int r = ti / nI;
  t.k = kbeg + r % nk;
  t.s = r / nk;
  return t;
}

template <bool kUpd, int kDen>
__global__ void __launch_bounds__(zv::THREADS, 1)
    k_tc_zvjp(Geo g, int u_bf16_bth, const void* __restrict__ u_rows, const __half* __restrict__ u16,
              const __nv_bfloat16* __restrict__ xraw, const float* __restrict__ ell,
              const float* __restrict__ lamlog, const __half* __restrict__ E, const void* __restrict__ dx32,
              const void* __restrict__ dv32, float* dell, float* dellend, __nv_bfloat16* dxo,
              __nv_bfloat16* dvo, int ntiles, int nI, int nk, int kbeg) {
  using namespace zv;
  constexpr bool den = kDen != 0;
  constexpr int NBT = 64 + kDen;     // E tiles per state
  constexpr int TOK = kUpd ? 128 : 256;
  constexpr int NBS = (NBT + TPS - 1) / TPS;   // B stages per work tile
  constexpr int NJ = (NBT + 1) / 2;            // A stages per work tile
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  if (pad > (uint32_t)SMEM_PAD) __trap();
  uint8_t* smem = smem_raw + pad;
  uint8_t* b_s = smem;
  uint32_t* xw2 = (uint32_t*)(b_s + NSB * TPS * TILE);   // [2 tiles][32 words][256]: scaled fp16 x
  uint32_t* uw2 = xw2 + 2 * 32 * NGEN;                    // [2 tiles][32 words][256]: scaled fp16 u
  uint32_t* dhw2 = uw2 + 2 * 32 * NGEN;                   // [2 tiles][256]: score-sum factor (dden | 1) pv
  uint64_t* bars = (uint64_t*)(dhw2 + 2 * NGEN);
  uint64_t* b_full = bars;
  uint64_t* b_empty = b_full + NSB;
  uint64_t* a_full = b_empty + NSB;
  uint64_t* a_empty = a_full + NSA;
  uint64_t* acc_full = a_empty + NSA;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* prep_full = acc_empty + 1;   // 2: a tile's operand words are ready (epilogue warps)
  uint64_t* prep_empty = prep_full + 2;  // 2: the generating warps are done with them
  uint32_t& tmem_base = *(uint32_t*)(prep_empty + 2);

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < NSB; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 2);   // one commit per MMA issuer
    }
    for (int i = 0; i < NSA; ++i) {
      mbar_init(&a_full[i], NGW);
      mbar_init(&a_empty[i], 1);
    }
    mbar_init(acc_full, 2);
    mbar_init(acc_empty, 8);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&prep_full[i], 8);
      mbar_init(&prep_empty[i], NGW);
    }
    fence_barrier_init();
  }
  if (w == W_TMA) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
#ifdef PA_TRACE
  const bool trc = blockIdx.x == 37;
#endif
  PA_TR6(trc && tid == 0, 0);

  if (w == W_TMA) {
    // four issuing lanes: a thread completes one copy per ~690 cycles whatever its
    // size (profiles/r01_bulk_copy_probe.txt); lane i copies E tile i of a stage
    if (l < 4) {
      int gb = 0;
      for (int it = 0, ti = blockIdx.x; ti < ntiles; ++it, ti += gridDim.x) {
        const ZvTile t = zv_tile(ti, nI, nk, kbeg);
        const uint8_t* Eb = (const uint8_t*)(E + (size_t)(t.s * g.nsl + t.k) * NBT * (TILE / 2));
        for (int m = 0; m < NBS; ++m, ++gb) {
          const int sb = gb % NSB;
          const int ntl = (m + 1) * TPS <= NBT ? TPS : NBT - m * TPS;
          if (gb >= NSB) mbar_wait(&b_empty[sb], ((gb / NSB) + 1) & 1);
          if (l == 0) mbar_expect_tx(&b_full[sb], ntl * TILE);
          __syncwarp(15u);
          if (l < ntl)
            bulk_load(b_s + (sb * TPS + l) * TILE, Eb + (size_t)(m * TPS + l) * TILE, TILE, &b_full[sb]);
        }
      }
    }
  } else if (w == W_MMA || w == W_MMA + 1) {
    // two issuers over alternating stages (global stage parity): one waits on its
    // barriers while the other's MMAs run.  Accumulators are zeroed by the
    // epilogue warps, so every MMA accumulates.
    const int mw = w - W_MMA;
    constexpr uint32_t idk = idesc_f16(128, 64, false, false);   // B K-major: N = c rows, K = e
    constexpr uint32_t idn = idesc_f16(128, 64, false, true);    // B MN-major: K = c rows, N = e
    const uint64_t bk0 = smem_desc(smem_u32(b_s), 16, 1024, 2);
    const uint64_t bn0 = smem_desc(smem_u32(b_s), 8192, 1024, 2);
    int gs0 = 0;
    for (int it = 0, ti = blockIdx.x; ti < ntiles; ++it, ti += gridDim.x, gs0 += NJ) {
      bool first = true;
      for (int j = 0; j < NJ; ++j) {
        const int gs = gs0 + j;
        // deterministic mode: w9 issues every stage in order (one summation order)
        if (g.det ? mw != 0 : (gs & 1) != mw) continue;
        if (first) {
          mbar_wait_w(acc_empty, it & 1);
          first = false;
        }
        const int m = (2 * j) / TPS, gb = it * NBS + m, sb = gb % NSB, sa = gs % NSA;
        mbar_wait_w(&b_full[sb], (gb / NSB) & 1);
        mbar_wait_w(&a_full[sa], (gs / NSA) & 1);
        PA_TR6(trc && it == 2 && l == 0, 300 + j);
        tc_fence_after();
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int jt = 2 * j + i;   // E tile
          if (jt >= NBT) break;
          const uint64_t to = (uint64_t)(((sb * TPS + jt % TPS) * TILE) >> 4);
          const uint32_t ab_t = tm + 128u + (uint32_t)(sa * 128 + i * 64);
          // group 0: query half 0 / update dk (K-major tile)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_ts_w(tm, ab_t + kk * 8, bk0 + to + (uint64_t)(kk * 2), idk, 1u);
          // group 1: query half 1 (K-major) / update dv (MN-major; nothing on the score-sum tile)
          if (!kUpd) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ts_w(tm + 64u, ab_t + 32u + kk * 8, bk0 + to + (uint64_t)(kk * 2), idk, 1u);
          } else if (jt < 64) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ts_w(tm + 64u, ab_t + 32u + kk * 8, bn0 + to + (uint64_t)(kk * 128), idn, 1u);
          }
        }
        tc_commit_w(&a_empty[sa]);
        {
          // each issuer releases the B stage after its last A stage in it (twice when
          // the B stage feeds a single A stage)
          const int jb = (m * TPS) / 2, je = ((m + 1) * TPS < NBT ? (m + 1) * TPS : NBT);
          const int jend = (je + 1) / 2;   // A stages [jb, jend)
          if (j + 2 >= jend) {
            tc_commit_w(&b_empty[sb]);
            if (jend - jb == 1) tc_commit_w(&b_empty[sb]);
          }
        }
      }
      if (!g.det) {
        tc_commit_w(acc_full);   // both issuers: count 2
      } else if (mw == 0) {
        tc_commit_w(acc_full);
        tc_commit_w(acc_full);
      }
    }
  } else if (w < NGW) {
    // generating threads: one token row per TMEM lane; the tile's scaled operand
    // words were prepared by the epilogue warps (off this critical path)
    const int gq = w >> 2, qd = w & 3;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    int gs0 = 0;
    for (int it = 0, ti = blockIdx.x; ti < ntiles; ++it, ti += gridDim.x, gs0 += NJ) {
      const int pb = it & 1;
      const uint32_t* xw = xw2 + pb * 32 * NGEN;
      PA_TR6(trc && it < 40 && tid == 0, 820 + it);
      mbar_wait(&prep_full[pb], (it >> 1) & 1);
      PA_TR6(trc && it < 40 && tid == 0, 860 + it);
      uint32_t vr[32];
      {
        const uint32_t* uw = uw2 + pb * 32 * NGEN;
#pragma unroll
        for (int i = 0; i < 32; ++i) vr[i] = uw[i * NGEN + tid];
      }
      const uint32_t dh = den ? dhw2[pb * NGEN + tid] : 0u;
      // the release of the next stage's A slot is tested while this stage's stores
      // drain (a blocking wait costs ~160 cycles even on a completed phase)
      bool nxt_ready = gs0 < NSA;
      for (int j = 0; j < NJ; ++j) {
        const int gs = gs0 + j, sa = gs % NSA;
        if (gs >= NSA && !__all_sync(0xffffffffu, nxt_ready)) mbar_wait(&a_empty[sa], ((gs / NSA) + 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int jt = 2 * j + i;   // E tile
          const uint32_t base = tm + lane_off + 128u + (uint32_t)(sa * 128 + i * 64 + gq * 32);
          if (jt < 64) {
            const uint32_t xb = xw[(jt >> 1) * NGEN + tid];
            const uint32_t bc = __byte_perm(xb, 0, (jt & 1) ? 0x3232 : 0x1010);
#pragma unroll
            {
              uint32_t o[32];
#pragma unroll
              for (int q = 0; q < 32; ++q) o[q] = hmul2_f16(bc, vr[q]);
              tmem_st32(base, o);
            }
          } else if (jt < NBT && (!kUpd || gq == 0)) {
            // score-sum tile E_G[c][b]: A_b = x_b * (dden | 1) pv
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t o[16];
#pragma unroll
              for (int q = 0; q < 16; ++q) o[q] = hmul2_f16(dh, xw[(h * 16 + q) * NGEN + tid]);
              tmem_st16(base + (uint32_t)(h * 16), o);
            }
          }
        }
        {
          const int g1 = gs + 1;
          nxt_ready = g1 < NSA || mbar_test_wait(&a_empty[g1 % NSA], ((g1 / NSA) + 1) & 1);
        }
        tc_wait_st();
        tc_fence_before();
        __syncwarp();
        if (l == 0) {
          mbar_arrive(&a_full[sa]);
          if (j == NJ - 1) mbar_arrive(&prep_empty[pb]);   // xw/uw of this tile are no longer read
        }
        PA_TR6(trc && it == 2 && tid == 0, 600 + j);
      }
    }
  } else if (w >= W_EPI && w < W_EPI + 8) {
    // epilogue warps: (1) prepare the operand words of tile it+2 (row loads from
    // HBM, power-of-two scales, fp16 conversion) while the MMAs of tile it+1 run;
    // (2) read tile it's accumulator, zero it and hand it back, add the fp32
    // intra-chunk part and store the final bf16 gradient rows
    const int e = w - W_EPI, gq = e >> 2, qd = w & 3, row = qd * 32 + l;
    const int pt = gq * 128 + row;   // column of this token in the operand words (= its generating thread)
    const int rr = kUpd ? row : gq * 128 + row;
    const bool u_is_x = kUpd && gq == 1;
    const bool ub = kUpd || u_bf16_bth;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    float fct_ring[2] = {0.f, 0.f};
    auto prepare = [&](int itp, int tip) {
      const int pb = itp & 1;
      if (itp >= 2) mbar_wait(&prep_empty[pb], ((itp >> 1) + 1) & 1);
      const ZvTile t = zv_tile(tip, nI, nk, kbeg);
      const bool live = t.I * TOK + rr < g.c;
      const int tok = t.k * g.c + t.I * TOK + (live ? rr : 0);
      const size_t xr = rowid(g, t.s, tok);
      uint32_t* xw = xw2 + pb * 32 * NGEN;
      uint32_t* uw = uw2 + pb * 32 * NGEN;
      const float lt = ell[(size_t)t.s * g.t + tok];
      const float lend = (kUpd && g.gated) ? lamlog[t.s * g.n + t.k] : 0.f;
      const float dsc = den ? (kUpd ? 1.f : __half2float(u16[((size_t)t.s * g.t + tok) * 16])) : 0.f;
      uint4 v8[8];
      const uint4* xg = (const uint4*)(xraw + xr * HD);
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) v8[c8] = xg[c8];
      float mx = 0.f;
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) mx = chunk_max(v8[c8], true, mx);
      // x (the bcast factor) and the vector operand u, both scaled by powers of two
      // into [1, 2) so fp16 products keep their precision for any input range
      const float px = pow2_norm(mx);
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        uint32_t o[4];
        chunk_f16(v8[c8], true, px, o);
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2) {
          xw[(c8 * 4 + e2) * NGEN + pt] = live ? o[e2] : 0u;
          if (u_is_x) uw[(c8 * 4 + e2) * NGEN + pt] = live ? o[e2] : 0u;
        }
      }
      float pv = px;
      if (!u_is_x) {
        const uint4* ug = ub ? (const uint4*)((const __nv_bfloat16*)u_rows + xr * HD)
                             : (const uint4*)((const __half*)u_rows + ((size_t)t.s * g.t + tok) * HD);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) v8[c8] = ug[c8];
        float mu = fabsf(dsc);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) mu = chunk_max(v8[c8], ub, mu);
        pv = pow2_norm(mu);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          uint32_t o[4];
          chunk_f16(v8[c8], ub, pv, o);
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) uw[(c8 * 4 + e2) * NGEN + pt] = o[e2];
        }
      }
      if (den) dhw2[pb * NGEN + pt] = pack_f16(dsc * pv, dsc * pv);
      // per-token factor: query c_m = sigma^2 gp_m, update W_j = exp(lend - ell_j);
      // dv counts each unordered pair twice (1/2); the operand scales come back here
      const float sscale =
          1.f / (kUpd ? pow2_neg_bits(g.ng - 1 - (g.k0 + t.k)) : pow2_neg_bits(g.k0 + t.k - 1));
      float fct = sscale * (kUpd ? (g.gated ? __expf(lend - lt) : 1.f) : g.scale * g.scale * __expf(lt));
      fct /= px * pv;
      if (u_is_x) fct *= 0.5f;
      if (pb) fct_ring[1] = fct; else fct_ring[0] = fct;
      __syncwarp();
      if (l == 0) mbar_arrive(&prep_full[pb]);
    };
    {
      uint32_t z[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
      for (int c = 0; c < 64; c += 16) tmem_st16(tm + lane_off + (uint32_t)(gq * 64 + c), z);
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (l == 0) mbar_arrive(acc_empty);
    }
    if (blockIdx.x < ntiles) prepare(0, blockIdx.x);
    if (blockIdx.x + gridDim.x < ntiles) prepare(1, blockIdx.x + gridDim.x);
    for (int it = 0, ti = blockIdx.x; ti < ntiles; ++it, ti += gridDim.x) {
      const ZvTile t = zv_tile(ti, nI, nk, kbeg);
      const bool live = t.I * TOK + rr < g.c;
      const int tok = t.k * g.c + t.I * TOK + rr;
      const bool is_dv = kUpd && gq == 1;
      const float fct = (it & 1) ? fct_ring[1] : fct_ring[0];
      mbar_wait(acc_full, it & 1);
      PA_TR6(trc && it < 40 && tid == W_EPI * 32, 900 + it);
      tc_fence_after();
      uint32_t r[64];
      const uint32_t acc = tm + lane_off + (uint32_t)(gq * 64);
      tmem_ld32(acc, r);
      tmem_ld32(acc + 32u, r + 32);
      tc_wait_ld();
      {
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
        for (int c = 0; c < 64; c += 16) tmem_st16(acc + (uint32_t)c, z);
      }
      tc_wait_st();
      tc_fence_before();
      __syncwarp();
      if (l == 0) mbar_arrive(acc_empty);
      if (live) {
        const size_t xr = rowid(g, t.s, tok);
        // intra-chunk part: fp32 rows (query side, reduce-added by the intra kernel)
        // or bf16 rows (update side)
        const size_t orow = ((size_t)t.s * g.t + tok) * HD;
        const float4* o32 = (const float4*)((const float*)dx32 + orow);
        const uint4* o16 = (const uint4*)((const __nv_bfloat16*)(is_dv ? dv32 : dx32) + orow);
        const uint4* xsrc = (const uint4*)(xraw + xr * HD);
        // the bf16 rows go out through shared memory: this tile's operand-word buffer
        // (xw2[it & 1]) is free once its accumulator is full (every generator read
        // of it precedes the last a_full arrival); 32 rows x 128 B per warp, 16-byte
        // chunks XOR-swizzled by row, then four whole 128-byte rows per warp store
        uint8_t* stg = (uint8_t*)(xw2 + (it & 1) * 32 * NGEN) + e * 4096;
        float c = 0.f, ci = 0.f;
#pragma unroll
        for (int a4 = 0; a4 < 8; a4 += 4) {
          float ov[4][8];
          uint4 xv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            if (kUpd) {
              const uint4 h8 = o16[a4 + i];
              const uint32_t* ph = (const uint32_t*)&h8;
#pragma unroll
              for (int e2 = 0; e2 < 4; ++e2) {
                const float2 f2 = __bfloat1622float2(*(const __nv_bfloat162*)&ph[e2]);
                ov[i][2 * e2] = f2.x;
                ov[i][2 * e2 + 1] = f2.y;
              }
            } else {
              const float4 v0 = o32[2 * (a4 + i)], v1 = o32[2 * (a4 + i) + 1];
              ov[i][0] = v0.x; ov[i][1] = v0.y; ov[i][2] = v0.z; ov[i][3] = v0.w;
              ov[i][4] = v1.x; ov[i][5] = v1.y; ov[i][6] = v1.z; ov[i][7] = v1.w;
            }
            if (!is_dv) xv[i] = xsrc[a4 + i];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int a = a4 + i;
            const float* f = (const float*)&r[a * 8];
            if (!is_dv) {
              const uint32_t* pxv = (const uint32_t*)&xv[i];
#pragma unroll
              for (int e2 = 0; e2 < 4; ++e2) {
                const float2 x2 = __bfloat1622float2(*(const __nv_bfloat162*)&pxv[e2]);
                c = fmaf(f[2 * e2], x2.x, fmaf(f[2 * e2 + 1], x2.y, c));
                if (!kUpd) ci = fmaf(ov[i][2 * e2], x2.x, fmaf(ov[i][2 * e2 + 1], x2.y, ci));
              }
            }
            const float* o = ov[i];
            *(uint4*)(stg + l * 128 + ((a ^ (l & 7)) << 4)) =
                make_uint4(pack_bf16(fmaf(f[0], fct, o[0]), fmaf(f[1], fct, o[1])),
                           pack_bf16(fmaf(f[2], fct, o[2]), fmaf(f[3], fct, o[3])),
                           pack_bf16(fmaf(f[4], fct, o[4]), fmaf(f[5], fct, o[5])),
                           pack_bf16(fmaf(f[6], fct, o[6]), fmaf(f[7], fct, o[7])));
          }
        }
        __syncwarp();
        {
          __nv_bfloat16* outp = is_dv ? dvo : dxo;
#pragma unroll
          for (int r4 = 0; r4 < 32; r4 += 4) {
            const int rw = r4 + (l >> 3), ch = l & 7;
            *(uint4*)(outp + rowid(g, t.s, tok - l + rw) * HD + ch * 8) =
                *(const uint4*)(stg + rw * 128 + ((ch ^ (rw & 7)) << 4));
          }
        }
        // d<., .>/d(log factor) = <dx~, x~>/2 (degree-2 homogeneity of phi'); the
        // intra-chunk query side follows the same way from the fp32 intra-chunk dq
        // rows (sum_j dP'_mj P_mj = <q_m, dq_m>/2; the intra-chunk kernel wrote the
        // key side; deterministic mode: the query-side pass added it instead)
        c *= 0.5f * fct;
        if (g.gated) {
          if (!kUpd) dell[(size_t)t.s * g.t + tok] += c + (g.det ? 0.f : 0.5f * ci);   // gp_m = exp(ell_m)
          else if (gq == 0) dellend[(size_t)t.s * g.t + tok] = c;   // suffix decay, finished in gate_finish
        }
      }
      PA_TR6(trc && it == 2 && tid == W_EPI * 32, 2);
      // the operand words of tile it+2 go into the buffer the eight epilogue warps
      // just staged tile it's rows through, and prepare() writes every warp's part
      // of it: all staging reads must be done first
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (ti + 2 * (int)gridDim.x < ntiles) prepare(it + 2, ti + 2 * gridDim.x);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == W_TMA) tmem_dealloc<512>(tm);
}

// chunk 0 without a prefix has no state query: dq is the intra-chunk part
// alone; its log-gate cotangent <q, dq>/2 as in the epilogue above
__global__ void __launch_bounds__(256) k_tc_dq_chunk0(Geo g, const float* __restrict__ dx32,
                                                      const __nv_bfloat16* __restrict__ xraw, float* dell,
                                                      __nv_bfloat16* dxo) {
  const int s = blockIdx.y;
  for (int i = blockIdx.x * 256 + threadIdx.x; i < g.c * 16; i += gridDim.x * 256) {
    const int r = i >> 4, c4 = (i & 15) * 4;
    const float4 v = *(const float4*)(dx32 + ((size_t)s * g.t + r) * HD + c4);
    const uint2 xq = *(const uint2*)(xraw + rowid(g, s, r) * HD + c4);
    const float2 x01 = __bfloat1622float2(*(const __nv_bfloat162*)&xq.x);
    const float2 x23 = __bfloat1622float2(*(const __nv_bfloat162*)&xq.y);
    float dot = v.x * x01.x + v.y * x01.y + v.z * x23.x + v.w * x23.y;
    // the 16 lanes (i & 15) of a row sit in one half-warp
#pragma unroll
    for (int o = 1; o < 16; o <<= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    *(uint2*)(dxo + rowid(g, s, r) * HD + c4) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
    if (g.gated && !g.det && (i & 15) == 0) dell[(size_t)s * g.t + r] += 0.5f * dot;
  }
}

int tc_zvjp(const Geo& g, bool upd, int u_bf16_bth, const void* u_rows, const __half* u16, const void* xraw,
            const float* ell, const float* lamlog, const __half* E, const void* dx32, const void* dv32,
            float* dell, float* dellend, void* dxo, void* dvo, cudaStream_t st) {
  using namespace zv;
  const int den = g.normalize ? 1 : 0;
  auto fn = upd ? (den ? k_tc_zvjp<true, 1> : k_tc_zvjp<true, 0>)
                : (den ? k_tc_zvjp<false, 1> : k_tc_zvjp<false, 0>);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int tok = upd ? 128 : 256;
  const int kbeg = (!upd && !g.prefix) ? 1 : 0;
  const int nI = (g.c + tok - 1) / tok, nk = g.n - kbeg;
  if (kbeg) {
    k_tc_dq_chunk0<<<dim3(8, g.ns), 256, 0, st>>>(g, (const float*)dx32, (const __nv_bfloat16*)xraw, dell,
                                                   (__nv_bfloat16*)dxo);
    count_launch();
  }
  const int ntiles = nI * nk * g.ns;
  if (ntiles <= 0) return 0;
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = ntiles < nsm ? ntiles : nsm;
  fn<<<grid, THREADS, SMEM, st>>>(g, u_bf16_bth, u_rows, u16, (const __nv_bfloat16*)xraw, ell, lamlog, E, dx32,
                                  dv32, dell, dellend, (__nv_bfloat16*)dxo, (__nv_bfloat16*)dvo, ntiles, nI, nk,
                                  kbeg);
  return 0;
}

}  // namespace pa
