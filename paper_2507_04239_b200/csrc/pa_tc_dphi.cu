// Token-major state VJP with the expand-VJP fused into the epilogue
// (reference gradients.py:46-76 expand_vjp, 191-213 update-state VJP,
// 406-431 query-state VJP), bf16/fp16 tcgen05 path, p = 2, d = e = 64.
//
//   query  (kUpd = false): dphi'(q~) = [dnum | dden] A'^T_{k-1}
//          -> dq = intra part + sigma^2 gp_m J^T dphi',  dell_m += <dq~, q~>/2
//   update (kUpd = true):  dphi'(k~) = [v | 1] dS~_k^T
//          -> dk = intra part + W_j J^T dphi',  cu_j = <dk~, k~>/2
//          and dv = intra part + W_j phi'(k_j) dS~_k (second GEMM)
//
// B200 design.  One CTA per 128-token tile.  The state (2304 feature slots x
// 64 columns, fp16) is streamed once, in 128-slot tiles: each tile feeds the
// dphi GEMM (M = 128 tokens, N = 128 slots, K = 64) and, on the update side,
// the dv GEMM (M = 128 tokens, N = 64, K = these 128 slots) from the same
// shared-memory stage (K-major for one, MN-major for the other), so the
// state is read from L2 once per CTA instead of twice.
// The expand-VJP loops over the 4x8 feature blocks with runtime block
// indices: each thread's x (its token row, fp32 and fp16) and dx live in
// shared memory (thread-private columns, conflict-free float4 rows) and the
// per-block working set (4 + 8 values of x, 8 dx accumulators of the current
// b-block) in registers.  The fully unrolled per-block code of the earlier
// kernel was ~140 KB of SASS and stalled on instruction fetch.
#include <cuda.h>

#include "pa_common.cuh"
#include "pa_sm100.cuh"
#include "pa_tc.cuh"
#include "pa_tc_common.cuh"

namespace pa {
using namespace sm100;
using namespace tc;

static __constant__ BlkTab c_blk_d = make_blk_tab();

#ifdef PA_TRACE
// debug build only (tools/trace_dphi.py): clock64 stamps of one CTA
__device__ long long g_trace3[512];
extern "C" int pa_debug_trace3(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trace3, sizeof(long long) * n);
}
#define PA_TR3(c, i) \
  if (c) g_trace3[(i)] = clock64()
#else
#define PA_TR3(c, i)
#endif

namespace dp2 {
constexpr int BM = 128 * 128;    // state stage: 128 slots x 64 fp16
constexpr int BD = 128 * 32;     // state stage score-sum part
constexpr int NST = 4;
constexpr int NT = FH / 128;     // 18 slot tiles
constexpr int XS = 16 * 128 * 16;   // fp32 x or dx: [16 float4][128 threads]
constexpr int XH = 8 * 128 * 16;    // fp16 x: [8 uint4][128 threads]
constexpr int AS = 128 * 128, AS16 = 128 * 32;   // query side: A rows staged in shared memory
constexpr int SMEM = 1024 + NST * (BM + BD) + 3 * XS + XH + AS + AS16 + 256;
// w0..w7 compute (two groups of four: group g owns the slot tiles nt = g mod 2,
// i.e. TMEM buffer g, and its own dx copy), w8 TMEM, w9 TMA, w10/w11 MMA
// (issuer m owns the tiles nt = m mod 2: each barrier wait costs ~160 cycles
// even when the phase is complete, so two issuers overlap their wait and
// commit latencies).  The issuing warps take the highest ids (the scheduler
// prefers high warp ids).
constexpr int THREADS = 384;
// TMEM columns (update side): dphi buffers [0, 256), dv accumulator [256, 320), A [320, 352),
// score-sum A [352, 360), generated phi'(k) buffers [384, 512); query side: 4 dphi buffers [0, 512)
constexpr uint32_t TA = 320, TA16 = 352;
constexpr int W_TMEM = 8, W_TMA = 9, W_MMA = 10;   // MMA issuers: w10, w11
}  // namespace dp2

__device__ __forceinline__ void load_row_f16_any(const __nv_bfloat16* src, uint32_t (&xp)[32]) {
  const uint4* row = (const uint4*)src;
#pragma unroll
  for (int c8 = 0; c8 < 8; ++c8) {
    const uint4 v4 = row[c8];
    const uint32_t* pv = (const uint32_t*)&v4;
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      const float2 f2 = __bfloat1622float2(*(const __nv_bfloat162*)&pv[e2]);
      xp[c8 * 4 + e2] = pack_f16(f2.x, f2.y);
    }
  }
}

struct ff2 {
  float x, y;
};
__device__ __forceinline__ ff2 ffma2(ff2 a, ff2 b, ff2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*(uint64_t*)&a), "l"(*(uint64_t*)&b), "l"(*(uint64_t*)&c));
  return *(ff2*)&r;
}

template <bool kUpd, int kDen>
__global__ void __launch_bounds__(dp2::THREADS, 1) k_tc_dphi2(
    const void* __restrict__ a_rows, int a_bf16_bth, const __half* __restrict__ a16_rows, Geo g,
    const __nv_bfloat16* __restrict__ xraw, const float* __restrict__ ell, const float* __restrict__ lamlog,
    const __half* __restrict__ b_main, const __half* __restrict__ b_den, const float* __restrict__ dx32,
    const float* __restrict__ dv32, float* dell, float* dellend, __nv_bfloat16* dxo, __nv_bfloat16* dvo) {
  using namespace dp2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* bm_s = smem;
  uint8_t* bd_s = bm_s + NST * BM;
  float4* x_s = (float4*)(bd_s + NST * BD);
  float4* dx_all = x_s + 16 * 128;          // [2 groups][16][128]
  uint4* xh_s = (uint4*)(dx_all + 2 * 16 * 128);
  uint8_t* as_s = (uint8_t*)(xh_s + 8 * 128);   // [128 tok][64] fp16 SW128 (query side)
  uint8_t* as16_s = as_s + AS;                    // [128 tok][16] fp16 SW32 (query side, normalize)
  uint64_t* bars = (uint64_t*)(as16_s + AS16);
  uint64_t* a_ready = bars;          // A operand in TMEM: 4 compute-warp arrivals
  uint64_t* b_full = a_ready + 1;    // NST
  uint64_t* b_empty = b_full + NST;  // NST
  // dphi TMEM buffers: update side 2 (TMEM also holds dv, phi'(k) and A), query
  // side 4 (A in shared memory): each compute group then owns two buffers, so
  // the MMA of its next tile overlaps its expand-VJP of the current one
  constexpr int NDB = kUpd ? 2 : 4;
  uint64_t* d_full = b_empty + NST;  // 4
  uint64_t* d_empty = d_full + 4;    // 4
  uint64_t* g_full = d_empty + 4;    // 2
  uint64_t* g_empty = g_full + 2;    // 2
  uint64_t* fin = g_empty + 2;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int I = blockIdx.x, k = blockIdx.y, s = blockIdx.z;
  const int tok0 = k * g.c + I * 128;
  constexpr bool den = kDen != 0;
  if (!kUpd && k == 0 && !g.prefix) {
    // chunk 0 has no state query: its dq is the intra-chunk part alone
    for (int i = tid; i < 128 * 16; i += THREADS) {
      const int r = i >> 4, c4 = (i & 15) * 4;
      const float4 v = *(const float4*)(dx32 + ((size_t)s * g.t + tok0 + r) * HD + c4);
      *(uint2*)(dxo + rowid(g, s, tok0 + r) * HD + c4) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
    }
    return;
  }
  // B operand: query side the state before chunk k (slot k), update side dS~_k;
  // undo their stored power-of-two scales
  const __half* bm = b_main + (size_t)(s * g.nsl + k) * ((size_t)FH * 64);
  const __half* bd = b_den + (size_t)(s * g.nsl + k) * ((size_t)FH * 16);
  const float sscale = 1.f / (kUpd ? pow2_neg_bits(g.ng - 1 - (g.k0 + k)) : pow2_neg_bits(g.k0 + k - 1));

  if (w == W_TMEM) tmem_alloc<512>(&tmem_base);
  if (tid == 0) {
    mbar_init(a_ready, 4);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&d_full[i], 1);
      mbar_init(&d_empty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&g_full[i], 4);
      mbar_init(&g_empty[i], 1);
    }
    mbar_init(fin, 2);
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  // TMEM: dphi buffers [0, 256), dv accumulator [256, 320), generated phi'(k) buffers [384, 512)

  if (w == W_TMA) {
    if (l == 0) {
      for (int nt = 0; nt < NT; ++nt) {
        const int st = nt % NST;
        if (nt >= NST) mbar_wait(&b_empty[st], ((nt / NST) + 1) & 1);
        mbar_expect_tx(&b_full[st], BM + (den ? BD : 0));
        bulk_load(bm_s + st * BM, bm + (size_t)nt * 128 * 64, BM, &b_full[st]);
        if (den) bulk_load(bd_s + st * BD, bd + (size_t)nt * 128 * 16, BD, &b_full[st]);
      }
    }
  } else if (w >= W_MMA) {
    {
      const int mw = w - W_MMA;
      constexpr uint32_t id128 = idesc_f16(128, 128, false, false);
      constexpr uint32_t id64mn = idesc_f16(128, 64, false, true);
      mbar_wait_w(a_ready, 0);
      tc_fence_after();
      // descriptors are built once; per-MMA work is a 64-bit add of (byte offset >> 4)
      const uint64_t bk0 = smem_desc(smem_u32(bm_s), 16, 1024, 2);      // K-major view of a state stage
      const uint64_t bn0 = smem_desc(smem_u32(bm_s), 8192, 1024, 2);    // MN-major view of the same stage
      const uint64_t bd0 = smem_desc(smem_u32(bd_s), 16, 256, 6);
      const uint64_t ak0 = smem_desc(smem_u32(as_s), 16, 1024, 2);
      const uint64_t a160 = smem_desc(smem_u32(as16_s), 16, 256, 6);
#ifdef PA_TRACE
      const bool trm = kUpd && blockIdx.x == 0 && blockIdx.y == 5 && blockIdx.z == 3 && mw == 0;
#endif
      PA_TR3(trm, 99);
      for (int nt = mw; nt < NT; nt += 2) {
        const int st = nt % NST, db = nt % NDB;
        mbar_wait_w(&b_full[st], (nt / NST) & 1);
        PA_TR3(trm, nt * 4 + 0);
        if (nt >= NDB) mbar_wait_w(&d_empty[db], ((nt / NDB) + 1) & 1);
        PA_TR3(trm, nt * 4 + 1);
        tc_fence_after();
        const uint64_t so = (uint64_t)((st * BM) >> 4);
        const uint32_t dt = tm + (uint32_t)(db * 128);
        if (kUpd) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ts_w(dt, tm + TA + (uint32_t)(kk * 8), bk0 + so + (uint64_t)(kk * 2), id128, kk > 0 ? 1u : 0u);
          if (den) mma_ts_w(dt, tm + TA16, bd0 + (uint64_t)((st * BD) >> 4), id128, 1u);
        } else {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            mma_ss_w(dt, ak0 + (uint64_t)(kk * 2), bk0 + so + (uint64_t)(kk * 2), id128, kk > 0 ? 1u : 0u);
          if (den) mma_ss_w(dt, a160, bd0 + (uint64_t)((st * BD) >> 4), id128, 1u);
        }
        tc_commit_w(&d_full[db]);
        PA_TR3(trm, 400 + nt);
        if (kUpd) {
          // dv += phi'(k) [128 tok x 128 slots] * dS~ tile [128 slots x 64] (same stage, MN-major)
          mbar_wait_w(&g_full[nt & 1], (nt >> 1) & 1);
          PA_TR3(trm, nt * 4 + 2);
          tc_fence_after();
          const uint32_t ab = tm + 384u + (uint32_t)((nt & 1) * 64);
          // both issuers accumulate into the zero-initialised dv columns
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) mma_ts_w(tm + 256u, ab + kk * 8, bn0 + so + (uint64_t)(kk * 128), id64mn, 1u);
          tc_commit_w(&g_empty[nt & 1]);
        }
        tc_commit_w(&b_empty[st]);
        PA_TR3(trm, nt * 4 + 3);
      }
      tc_commit_w(fin);
    }
  } else if (w < 8) {
    const int q = w & 3, grp = w >> 2, row = q * 32 + l;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int tok = tok0 + row;
    const float lt = ell[(size_t)s * g.t + tok];
    float4* dx_s = dx_all + grp * (16 * 128);
    // phi' is generated from the exact bf16 row; the per-token factor
    //   query : c_m = sigma^2 gp_m        (y_state = c_m phi'(q) A')
    //   update: W_j = exp(lend - ell_j)   (S' = sum_j W_j phi'(k_j) u_j^T)
    // multiplies the fp32 results instead of a rounded operand.
    const float fct =
        sscale * (kUpd ? (g.gated ? __expf(lamlog[s * g.n + k] - lt) : 1.f) : g.scale * g.scale * __expf(lt));
#pragma unroll
    for (int i = 0; i < 16; ++i) dx_s[i * 128 + row] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (grp == 0) {
      // stage this token's row: fp32 x (thread-private float4 columns) and fp16 x
      const uint4* src = (const uint4*)(xraw + rowid(g, s, tok) * HD);
#pragma unroll
      for (int c8 = 0; c8 < 8; ++c8) {
        const uint4 v4 = src[c8];
        const uint32_t* pv = (const uint32_t*)&v4;
        float f[8];
#pragma unroll
        for (int e2 = 0; e2 < 4; ++e2) {
          const float2 f2 = __bfloat1622float2(*(const __nv_bfloat162*)&pv[e2]);
          f[2 * e2] = f2.x;
          f[2 * e2 + 1] = f2.y;
        }
        x_s[(2 * c8) * 128 + row] = make_float4(f[0], f[1], f[2], f[3]);
        x_s[(2 * c8 + 1) * 128 + row] = make_float4(f[4], f[5], f[6], f[7]);
        if (kUpd)
          xh_s[c8 * 128 + row] =
              make_uint4(pack_f16(f[0], f[1]), pack_f16(f[2], f[3]), pack_f16(f[4], f[5]), pack_f16(f[6], f[7]));
      }
    }
    if (grp == 0) {
      // the A operand of the dphi GEMM goes to TMEM (one row per lane): the MMA then
      // reads only the state tile from shared memory
      uint32_t ar[32];
      if (a_bf16_bth) {
        // bf16 rows in the reference layout, converted to fp16 pairs (exact for |x| < 65504)
        load_row_f16_any((const __nv_bfloat16*)a_rows + rowid(g, s, tok) * HD, ar);
      } else {
        const uint4* src = (const uint4*)((const __half*)a_rows + ((size_t)s * g.t + tok) * HD);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) *(uint4*)&ar[c8 * 4] = src[c8];
      }
      if (kUpd) {
        tmem_st16(tm + TA + lane_off, ar);
        tmem_st16(tm + TA + 16 + lane_off, ar + 16);
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
#pragma unroll
        for (int c = 0; c < 64; c += 16) tmem_st16(tm + 256u + lane_off + c, z);   // dv accumulator
      } else {
        // K-major SW128 row of the shared-memory A tile
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) *(uint4*)(as_s + sw128_off(row, c8)) = *(const uint4*)&ar[c8 * 4];
      }
      if (den) {
        uint32_t a16[8];
        if (kUpd) {
          // [v | 1]: column 0 = 1
          a16[0] = pack_f16(1.f, 0.f);
#pragma unroll
          for (int i = 1; i < 8; ++i) a16[i] = 0u;
          tmem_st8(tm + TA16 + lane_off, a16);
        } else {
          const uint4* s16 = (const uint4*)(a16_rows + ((size_t)s * g.t + tok) * 16);
          // SW32 row: 16-byte chunk c at ((c ^ ((row >> 2) & 1)) << 4)
          const uint32_t xr = ((uint32_t)row >> 2) & 1u;
          *(uint4*)(as16_s + row * 32 + ((0u ^ xr) << 4)) = s16[0];
          *(uint4*)(as16_s + row * 32 + ((1u ^ xr) << 4)) = s16[1];
        }
      }
      if (!kUpd) fence_async_smem();
      tc_wait_st();
      tc_fence_before();
    }
    __syncwarp();
    if (grp == 0 && l == 0) mbar_arrive(a_ready);
    asm volatile("bar.sync 1, 256;" ::: "memory");   // x staged for both groups

    // generate phi'(k~) for the 128 slots of tile nt into TMEM buffer nt % 2
#ifdef PA_TRACE
    const bool trc = kUpd && blockIdx.x == 0 && blockIdx.y == 5 && blockIdx.z == 3 && (w & 3) == 0 && l == 0;
#endif
    auto gen = [&](int nt) {
      const int db = nt & 1;
      PA_TR3(trc, 300 + nt * 3 + 0);
      if (nt >= 2) mbar_wait(&g_empty[db], ((nt >> 1) + 1) & 1);
      PA_TR3(trc, 300 + nt * 3 + 1);
      const uint32_t gb = tm + 384u + (uint32_t)(db * 64) + lane_off;
#pragma unroll
      for (int cb = 0; cb < 4; ++cb) {
        const int blk = nt * 4 + cb, al = c_blk_d.al[blk], be = c_blk_d.be[blk];
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
        tmem_st16(gb + (uint32_t)(cb * 16), o);
      }
      tc_wait_st();
      PA_TR3(trc, 300 + nt * 3 + 2);
      tc_fence_before();
      __syncwarp();
      if (l == 0) mbar_arrive(&g_full[db]);
    };

    if (kUpd) gen(grp);
    ff2 dxb[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};   // dx of the current b-block (8 dims)
    int cur_be = 0;
    float4 xb0 = x_s[0 * 128 + row], xb1 = x_s[1 * 128 + row];
    auto flush_b = [&](int be) {
      float4 d0 = dx_s[(2 * be) * 128 + row], d1 = dx_s[(2 * be + 1) * 128 + row];
      d0.x += dxb[0].x;
      d0.y += dxb[0].y;
      d0.z += dxb[1].x;
      d0.w += dxb[1].y;
      d1.x += dxb[2].x;
      d1.y += dxb[2].y;
      d1.z += dxb[3].x;
      d1.w += dxb[3].y;
      dx_s[(2 * be) * 128 + row] = d0;
      dx_s[(2 * be + 1) * 128 + row] = d1;
    };
    for (int nt = grp; nt < NT; nt += 2) {
      PA_TR3(trc, 100 + nt * 4 + 0);
      const int db = nt % NDB;
      PA_TR3(trc, 100 + nt * 4 + 1);
      mbar_wait(&d_full[db], (nt / NDB) & 1);
      PA_TR3(trc, 100 + nt * 4 + 2);
      tc_fence_after();
      const uint32_t dt = tm + (uint32_t)(db * 128) + lane_off;
      // 8 half-blocks (16 columns: a-rows 2hh, 2hh+1 of a 4x8 block); the TMEM load
      // of half-block u+1 is in flight while u is processed (a load round trip
      // costs ~130 cycles, tools/tmem_rate.cu)
      uint32_t gbuf[2][16];
      tmem_ld16(dt, gbuf[0]);
      float dxa[4];
      float4 xa = make_float4(0.f, 0.f, 0.f, 0.f);
      int al = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int cb = u >> 1, hh = u & 1;
        if (hh == 0) {
          const int blk = nt * 4 + cb, be = c_blk_d.be[blk];
          al = c_blk_d.al[blk];
          if (be != cur_be) {
            flush_b(cur_be);
            cur_be = be;
            dxb[0] = dxb[1] = dxb[2] = dxb[3] = ff2{0.f, 0.f};
            xb0 = x_s[(2 * be) * 128 + row];
            xb1 = x_s[(2 * be + 1) * 128 + row];
          }
          xa = x_s[al * 128 + row];
        }
        tc_wait_ld();
        if (u + 1 < 8) tmem_ld16(dt + (uint32_t)((u + 1) * 16), gbuf[(u + 1) & 1]);
        const uint32_t* gr = gbuf[u & 1];
        const float xav[4] = {xa.x, xa.y, xa.z, xa.w};
        const ff2 xbp[4] = {{xb0.x, xb0.y}, {xb0.z, xb0.w}, {xb1.x, xb1.y}, {xb1.z, xb1.w}};
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int ia = 2 * hh + i;
          const ff2 xai = {xav[ia], xav[ia]};
          ff2 t = {0.f, 0.f};
#pragma unroll
          for (int jp = 0; jp < 4; ++jp) {
            const ff2 gg = {__uint_as_float(gr[i * 8 + 2 * jp]), __uint_as_float(gr[i * 8 + 2 * jp + 1])};
            dxb[jp] = ffma2(gg, xai, dxb[jp]);   // dx[b] += g x[a]
            t = ffma2(gg, xbp[jp], t);           // dx[a] += g x[b]
          }
          dxa[ia] = t.x + t.y;
        }
        if (hh == 1) {
          float4 da = dx_s[al * 128 + row];
          da.x += dxa[0];
          da.y += dxa[1];
          da.z += dxa[2];
          da.w += dxa[3];
          dx_s[al * 128 + row] = da;
        }
      }
      PA_TR3(trc, 100 + nt * 4 + 3);
      tc_fence_before();
      __syncwarp();
      if (l == 0) mbar_arrive(&d_empty[db]);
      if (kUpd && nt + 2 < NT) gen(nt + 2);
    }
    flush_b(cur_be);
    PA_TR3(trc, 200);
    asm volatile("bar.sync 1, 256;" ::: "memory");   // both dx copies complete

    // epilogue: group 0 writes the final gradient rows (intra-chunk part + state
    // part, stored once in bf16); group 1 the dv rows on the update side
    float c = 0.f;
    if (grp == 0) {
      const float4* dx1 = dx_all + 16 * 128;
      const float* o = dx32 + ((size_t)s * g.t + tok) * HD;
      uint4* dst = (uint4*)(dxo + rowid(g, s, tok) * HD);
#pragma unroll
      for (int a8 = 0; a8 < 8; ++a8) {
        float4 d0 = dx_s[(2 * a8) * 128 + row], d1 = dx_s[(2 * a8 + 1) * 128 + row];
        const float4 e0 = dx1[(2 * a8) * 128 + row], e1 = dx1[(2 * a8 + 1) * 128 + row];
        d0 = make_float4(d0.x + e0.x, d0.y + e0.y, d0.z + e0.z, d0.w + e0.w);
        d1 = make_float4(d1.x + e1.x, d1.y + e1.y, d1.z + e1.z, d1.w + e1.w);
        const float4 x0 = x_s[(2 * a8) * 128 + row], x1 = x_s[(2 * a8 + 1) * 128 + row];
        c += d0.x * x0.x + d0.y * x0.y + d0.z * x0.z + d0.w * x0.w + d1.x * x1.x + d1.y * x1.y + d1.z * x1.z +
             d1.w * x1.w;
        const float4 v0 = *(const float4*)(o + a8 * 8), v1 = *(const float4*)(o + a8 * 8 + 4);
        dst[a8] = make_uint4(pack_bf16(fmaf(d0.x, fct, v0.x), fmaf(d0.y, fct, v0.y)),
                             pack_bf16(fmaf(d0.z, fct, v0.z), fmaf(d0.w, fct, v0.w)),
                             pack_bf16(fmaf(d1.x, fct, v1.x), fmaf(d1.y, fct, v1.y)),
                             pack_bf16(fmaf(d1.z, fct, v1.z), fmaf(d1.w, fct, v1.w)));
      }
    }
    c *= 0.5f * fct;   // = d<.,.>/d(log factor): degree-2 homogeneity of phi'
    if (!kUpd) {
      if (grp == 0 && g.gated) dell[(size_t)s * g.t + tok] += c;   // gp_m = exp(ell_m)
    } else if (grp == 0) {
      // suffix-decay cotangent: -c on ell_tok and +c on ell_end; summed over the
      // chunk this is an exclusive prefix sum (no cancellation), done in gate_finish
      if (g.gated) dellend[(size_t)s * g.t + tok] = c;
    } else {
      PA_TR3(trc, 201);
      mbar_wait(fin, 0);
      PA_TR3(trc, 202);
      tc_fence_after();
      uint32_t r[64];
      tmem_ld32(tm + 256u + lane_off, r);
      tmem_ld32(tm + 256u + lane_off + 32, r + 32);
      tc_wait_ld();
      const float* ov = dv32 + ((size_t)s * g.t + tok) * HD;
      uint4* dst = (uint4*)(dvo + rowid(g, s, tok) * HD);
#pragma unroll
      for (int a = 0; a < 64; a += 8) {
        const float4 v0 = *(const float4*)(ov + a), v1 = *(const float4*)(ov + a + 4);
        float f[8];
#pragma unroll
        for (int z = 0; z < 8; ++z) f[z] = __uint_as_float(r[a + z]) * fct;
        dst[a / 8] = make_uint4(pack_bf16(f[0] + v0.x, f[1] + v0.y), pack_bf16(f[2] + v0.z, f[3] + v0.w),
                                pack_bf16(f[4] + v1.x, f[5] + v1.y), pack_bf16(f[6] + v1.z, f[7] + v1.w));
      }
    }
  }
  if (w < 8) mbar_wait(fin, 0);   // the MMA stream must drain before TMEM is released
  tc_fence_before();
  __syncthreads();
  if (w == W_TMEM) tmem_dealloc<512>(tm);
}

int tc_dphi(const Geo& g, bool upd, const void* a_rows, int a_bf16_bth, const __half* a16_rows, const void* xraw,
            const float* ell, const float* lamlog, const __half* b_main, const __half* b_den, const float* dx32,
            const float* dv32, float* dell, float* dellend, void* dxo, void* dvo, cudaStream_t st) {
  using namespace dp2;
  const int den = g.normalize ? 1 : 0;
  auto fn = upd ? (den ? k_tc_dphi2<true, 1> : k_tc_dphi2<true, 0>)
                : (den ? k_tc_dphi2<false, 1> : k_tc_dphi2<false, 0>);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  fn<<<dim3(g.c / 128, g.n, g.ns), THREADS, SMEM, st>>>(a_rows, a_bf16_bth, a16_rows, g, (const __nv_bfloat16*)xraw, ell, lamlog,
                                                         b_main, b_den, dx32, dv32, dell, dellend,
                                                         (__nv_bfloat16*)dxo, (__nv_bfloat16*)dvo);
  return 0;
}

}  // namespace pa
