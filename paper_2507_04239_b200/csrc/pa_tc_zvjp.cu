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
// w8 TMA (E tiles); w19 TMA (token rows, one tile ahead); w9/w10 MMA issuers
// over alternating stages; w11..w18 epilogue.  TMEM: one accumulator [0, 128), zeroed and handed back by
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

#ifndef ZV_EXPERIMENT
#define ZV_EXPERIMENT 0
#endif
namespace zv {
constexpr int TILE = 64 * 128;   // bytes of one E tile: 64 rows (c) x 64 fp16 (e), SW128
constexpr int NSB = 3;           // B ring: 4 E tiles (32 KB, one bulk copy) per stage
constexpr int TPS = 4;           // E tiles per B stage
constexpr int NSA = 3;           // A stages in TMEM (two E tiles each)
constexpr int NGEN = 256;        // token rows per tile (x words are kept per row)
constexpr int NGW = 8;           // generating warps: 2 groups x 4 lane quadrants
constexpr int THREADS = 640;
constexpr int W_TMA = 8, W_MMA = 9, W_EPI = 11, W_ROWS = 19;   // MMA issuers: w9 (even stages), w10 (odd stages)
constexpr int ROWS = 256 * 128;  // token rows of one operand (up to 256 tokens, bf16, SW128)
constexpr int XW = 32 * NGEN * 4;   // fp16 x words, [word][thread]
constexpr int SMEM = 1024 + NSB * TPS * TILE + 2 * ROWS + XW + 4 * 256 * 4 + 16 + 512;
}  // namespace zv

// 2^-floor(log2(m)) for m > 0 (so m * p in [1, 2)), 1 for m == 0
__device__ __forceinline__ float pow2_norm(float m) {
  if (!(m > 0.f)) return 1.f;
  const int e = ((__float_as_int(m) >> 23) & 255) - 127;
  return __int_as_float((127 - e) << 23);
}

// 64 bf16 (or fp16) values: max |x|, and fp16x2 words scaled by p (a power of two)
__device__ __forceinline__ float row_max(const uint4 (&src)[8], bool is_bf16) {
  float m = 0.f;
#pragma unroll
  for (int c8 = 0; c8 < 8; ++c8) {
    const uint32_t* pv = (const uint32_t*)&src[c8];
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      const float2 f2 = is_bf16 ? __bfloat1622float2(*(const __nv_bfloat162*)&pv[e2])
                                : __half22float2(*(const __half2*)&pv[e2]);
      m = fmaxf(m, fmaxf(fabsf(f2.x), fabsf(f2.y)));
    }
  }
  return m;
}
__device__ __forceinline__ void row_f16(const uint4 (&src)[8], bool is_bf16, float p, uint32_t (&o)[32]) {
#pragma unroll
  for (int c8 = 0; c8 < 8; ++c8) {
    const uint32_t* pv = (const uint32_t*)&src[c8];
#pragma unroll
    for (int e2 = 0; e2 < 4; ++e2) {
      const float2 f2 = is_bf16 ? __bfloat1622float2(*(const __nv_bfloat162*)&pv[e2])
                                : __half22float2(*(const __half2*)&pv[e2]);
      o[c8 * 4 + e2] = pack_f16(f2.x * p, f2.y * p);
    }
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
    k_tc_zvjp(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_u, Geo g,
              int u_bf16_bth, const __half* __restrict__ u16, const __nv_bfloat16* __restrict__ xraw,
              const float* __restrict__ ell, const float* __restrict__ lamlog, const __half* __restrict__ E,
              const float* __restrict__ dx32, const float* __restrict__ dv32, float* dell, float* dellend,
              __nv_bfloat16* dxo, __nv_bfloat16* dvo, int ntiles, int nI, int nk, int kbeg) {
  using namespace zv;
  constexpr bool den = kDen != 0;
  constexpr int NBT = 64 + kDen;     // E tiles per state = stages per tile
  constexpr int TOK = kUpd ? 128 : 256;
  constexpr int NBOX = TOK / 128;
  constexpr int NBS = (NBT + TPS - 1) / TPS;   // B stages per work tile
  constexpr int NJ = (NBT + 1) / 2;            // A stages per work tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* b_s = smem;
  uint8_t* xrow_s = b_s + NSB * TPS * TILE;
  uint8_t* urow_s = xrow_s + ROWS;
  uint32_t* xw = (uint32_t*)(urow_s + ROWS);
  float* meta = (float*)(xw + 32 * NGEN);   // [2][256] per-token factor
  float* scal = meta + 2 * 256;             // [2][256] this tile's ell, dden (loaded with the rows) + lamlog
  uint64_t* bars = (uint64_t*)(scal + 2 * 256 + 4);
  uint64_t* b_full = bars;
  uint64_t* b_empty = b_full + NSB;
  uint64_t* a_full = b_empty + NSB;
  uint64_t* a_empty = a_full + NSA;
  uint64_t* acc_full = a_empty + NSA;
  uint64_t* acc_empty = acc_full + 1;
  uint64_t* meta_full = acc_empty + 1;  // 2
  uint64_t* meta_empty = meta_full + 2; // 2
  uint64_t* rows_full = meta_empty + 2;
  uint64_t* rows_empty = rows_full + 1;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  if (tid == 0) {
    for (int i = 0; i < NSB; ++i) {
      mbar_init(&b_full[i], 1);
      mbar_init(&b_empty[i], 2);   // one commit per MMA issuer
    }
    for (int i = 0; i < NSA; ++i) {
      mbar_init(&a_full[i], 8);
      mbar_init(&a_empty[i], 1);
    }
    mbar_init(acc_full, 2);
    mbar_init(acc_empty, 8);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&meta_full[i], 8);
      mbar_init(&meta_empty[i], 8);
    }
    mbar_init(rows_full, 2);   // TMA bytes + the loader warp's scalar stores
    mbar_init(rows_empty, NGW);
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
    // and row box i of a tile
    if (l < 4) {
      int gb = 0;
      for (int it = 0, ti = blockIdx.x; ti < ntiles; ++it, ti += gridDim.x) {
        const ZvTile t = zv_tile(ti, nI, nk, kbeg);
        const uint8_t* Eb = (const uint8_t*)(E + (size_t)(t.s * g.nsl + t.k) * NBT * (TILE / 2));
        for (int m = 0; m < NBS; ++m, ++gb) {
          const int sb = gb % NSB;
          const int ntl = (m + 1) * TPS <= NBT ? TPS : NBT - m * TPS;
          if (gb >= NSB) mbar_wait(&b_empty[sb], ((gb / NSB) + 1) & 1);
          PA_TR6(trc && it == 2 && l == 0, 100 + m);
          if (l == 0) mbar_expect_tx(&b_full[sb], ntl * TILE);
          __syncwarp(15u);
          if (l < ntl)
            bulk_load(b_s + (sb * TPS + l) * TILE, Eb + (size_t)(m * TPS + l) * TILE, TILE, &b_full[sb]);
        }
      }
    }
  } else if (w == W_ROWS) {
    // token rows, one tile ahead of the generating warps (single buffer: they
    // release it as soon as their rows are in registers), in its own warp so the
    // next tile's rows do not queue behind this tile's E stream; the tile's
    // per-token scalars go to shared memory with them (loaded by the generating
    // warps themselves, their HBM latency sat in every tile prologue)
    for (int it = 0, ti = blockIdx.x; ti < ntiles; ++it, ti += gridDim.x) {
      const ZvTile t = zv_tile(ti, nI, nk, kbeg);
      const int tok0 = t.k * g.c + t.I * TOK;
      const int bi = t.s / g.h, hi = t.s - bi * g.h;
      if (it >= 1) mbar_wait(rows_empty, (it - 1) & 1);
      __syncwarp();
      if (l == 0) mbar_expect_tx(rows_full, 2 * TOK * 128);
      __syncwarp();
      if (l < 2 * NBOX) {
        const int bx = l >> 1;
        if ((l & 1) == 0)
          tma_load_4d(xrow_s + bx * 16384, &tm_x, rows_full, 0, hi, tok0 + bx * 128, bi);
        else if (kUpd || u_bf16_bth)
          tma_load_4d(urow_s + bx * 16384, &tm_u, rows_full, 0, hi, tok0 + bx * 128, bi);
        else
          tma_load_2d(urow_s + bx * 16384, &tm_u, rows_full, 0, t.s * g.t + tok0 + bx * 128);
      }
      for (int i = l; i < TOK; i += 32) {
        const bool in = t.I * TOK + i < g.c;
        scal[i] = in ? ell[(size_t)t.s * g.t + tok0 + i] : 0.f;
        if (den && !kUpd) scal[256 + i] = in ? __half2float(u16[((size_t)t.s * g.t + tok0 + i) * 16]) : 0.f;
      }
      if (l == 0) scal[512] = (kUpd && g.gated) ? lamlog[t.s * g.n + t.k] : 0.f;
      __syncwarp();
      if (l == 0) mbar_arrive(rows_full);
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
#ifdef PA_TRACE
    long long wb = 0, wa = 0, wi = 0, we = 0;
#endif
    for (int it = 0, ti = blockIdx.x; ti < ntiles; ++it, ti += gridDim.x, gs0 += NJ) {
      bool first = true;
      for (int j = 0; j < NJ; ++j) {
        const int gs = gs0 + j;
        if ((gs & 1) != mw) continue;
        if (first) {
#ifdef PA_TRACE
          long long c9 = clock64();
#endif
          mbar_wait_w(acc_empty, it & 1);
#ifdef PA_TRACE
          we += clock64() - c9;
#endif
          first = false;
        }
        const int m = (2 * j) / TPS, gb = it * NBS + m, sb = gb % NSB, sa = gs % NSA;
#ifdef PA_TRACE
        long long c0 = clock64();
#endif
        mbar_wait_w(&b_full[sb], (gb / NSB) & 1);
#ifdef PA_TRACE
        long long c1 = clock64();
        wb += c1 - c0;
#endif
        PA_TR6(trc && it == 2 && l == 0, 200 + j);
        mbar_wait_w(&a_full[sa], (gs / NSA) & 1);
#ifdef PA_TRACE
        long long c2 = clock64();
        wa += c2 - c1;
#endif
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
        PA_TR6(trc && it == 2 && l == 0, 400 + j);
#ifdef PA_TRACE
        wi += clock64() - c2;
#endif
      }
      tc_commit_w(acc_full);   // both issuers: count 2
    }
#ifdef PA_TRACE
    if (trc && l == 0) {
      g_trace6[(kUpd ? 0 : 1024) + 700 + mw * 4 + 0] = wb;
      g_trace6[(kUpd ? 0 : 1024) + 700 + mw * 4 + 1] = wa;
      g_trace6[(kUpd ? 0 : 1024) + 700 + mw * 4 + 2] = wi;
      g_trace6[(kUpd ? 0 : 1024) + 700 + mw * 4 + 3] = we;
    }
#endif
  } else if (w < NGW) {
    // generating threads: one token row per TMEM lane
    const int gq = w >> 2, qd = w & 3, row = qd * 32 + l;
    const int xt = tid;   // this token's column in xw
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    const bool u_is_x = kUpd && gq == 1;
    const bool ub = kUpd || u_bf16_bth;
    const int rr = kUpd ? row : gq * 128 + row;   // row in the tile's row buffers
    const uint32_t roff = (uint32_t)(rr >> 7) * 16384u + (uint32_t)(rr & 127) * 128u;
#ifdef PA_TRACE
    long long gw = 0, gp = 0, gr = 0, gm = 0;
#endif
    int gs0 = 0;
    for (int it = 0, ti = blockIdx.x; ti < ntiles; ++it, ti += gridDim.x, gs0 += NJ) {
      const ZvTile t = zv_tile(ti, nI, nk, kbeg);
      const int ab = it & 1;
      const bool live = t.I * TOK + rr < g.c;
      // undo the stored power-of-two scale of the state
      const float sscale =
          1.f / (kUpd ? pow2_neg_bits(g.ng - 1 - (g.k0 + t.k)) : pow2_neg_bits(g.k0 + t.k - 1));
      uint32_t vr[32];
      float px, pv, lt, lend, dsc;
      PA_TR6(trc && it == 5 && tid == 0, 805);
      PA_TR6(trc && it == 4 && tid == 0, 806);
#ifdef PA_TRACE
      long long cp0 = clock64();
#endif
      {
        mbar_wait(rows_full, it & 1);
#ifdef PA_TRACE
        gr += clock64() - cp0;
#endif
        PA_TR6(trc && it == 5 && tid == 0, 800);
        lt = scal[rr];
        lend = scal[512];
        dsc = (den && !kUpd) ? scal[256 + rr] : (kUpd ? 1.f : 0.f);
        // two passes over each shared-memory row (max, then scaled conversion) keep
        // the register footprint at the 32 words of u: holding both rows and their
        // conversions spilled and cost ~7K cycles per tile
        auto chunk = [&](const uint8_t* base, int c8) {
          return *(const uint4*)(base + roff + (((uint32_t)c8 ^ (uint32_t)(rr & 7)) << 4));
        };
        auto chunk_max = [&](uint4 v4, bool is_bf16, float m) {
          const uint32_t* pv4 = (const uint32_t*)&v4;
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            const float2 f2 = is_bf16 ? __bfloat1622float2(*(const __nv_bfloat162*)&pv4[e2])
                                      : __half22float2(*(const __half2*)&pv4[e2]);
            m = fmaxf(m, fmaxf(fabsf(f2.x), fabsf(f2.y)));
          }
          return m;
        };
        auto chunk_f16 = [&](uint4 v4, bool is_bf16, float p, uint32_t* o) {
          const uint32_t* pv4 = (const uint32_t*)&v4;
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            const float2 f2 = is_bf16 ? __bfloat1622float2(*(const __nv_bfloat162*)&pv4[e2])
                                      : __half22float2(*(const __half2*)&pv4[e2]);
            o[e2] = pack_f16(f2.x * p, f2.y * p);
          }
        };
        // one row at a time in registers (max, then scaled conversion): a separate
        // max pass over shared memory cost ~10K cycles per tile, holding both rows
        // and their conversions spilled
        uint4 v8[8];
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) v8[c8] = chunk(xrow_s, c8);
        float mx = 0.f;
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) mx = chunk_max(v8[c8], true, mx);
        // x (the bcast factor) and the vector operand u, both scaled by powers of two
        // into [1, 2) so fp16 products keep their precision for any input range
        px = pow2_norm(mx);
#pragma unroll
        for (int c8 = 0; c8 < 8; ++c8) {
          uint32_t o[4];
          chunk_f16(v8[c8], true, px, o);
#pragma unroll
          for (int e2 = 0; e2 < 4; ++e2) {
            xw[(c8 * 4 + e2) * NGEN + xt] = live ? o[e2] : 0u;
            if (u_is_x) vr[c8 * 4 + e2] = live ? o[e2] : 0u;
          }
        }
        if (u_is_x) {
          pv = px;
        } else {
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) v8[c8] = chunk(urow_s, c8);
          float mu = fabsf(dsc);
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) mu = chunk_max(v8[c8], ub, mu);
          pv = pow2_norm(mu);
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) chunk_f16(v8[c8], ub, pv, &vr[c8 * 4]);
        }
        PA_TR6(trc && it == 5 && tid == 0, 801);
        __syncwarp();
        if (l == 0) mbar_arrive(rows_empty);
        PA_TR6(trc && it == 5 && tid == 0, 802);
      }
      // per-token factor for the epilogue: query c_m = sigma^2 gp_m, update
      // W_j = exp(lend - ell_j); dv counts each unordered pair twice (1/2)
      float fct = sscale * (kUpd ? (g.gated ? __expf(lend - lt) : 1.f) : g.scale * g.scale * __expf(lt));
      fct /= px * pv;
      if (kUpd && gq == 1) fct *= 0.5f;
#ifdef PA_TRACE
      long long cm0 = clock64();
#endif
      PA_TR6(trc && it == 5 && tid == 0, 803);
      if (it >= 2) mbar_wait(&meta_empty[ab], ((it >> 1) + 1) & 1);   // the epilogue of tile it-2 has read its factors
      PA_TR6(trc && it == 5 && tid == 0, 804);
#ifdef PA_TRACE
      gm += clock64() - cm0;
#endif
      meta[ab * 256 + gq * 128 + row] = fct;
      __syncwarp();
      if (l == 0) mbar_arrive(&meta_full[ab]);
#ifdef PA_TRACE
      gp += clock64() - cp0;
#endif
      PA_TR6(trc && it == 5 && tid == 0, 807);

      // the release of the next stage's A slot is tested while this stage's stores
      // drain (a blocking wait costs ~160 cycles even on a completed phase)
      bool nxt_ready = gs0 < NSA;
      for (int j = 0; j < NJ; ++j) {
        const int gs = gs0 + j, sa = gs % NSA;
#ifdef PA_TRACE
        long long c0 = clock64();
#endif
        if (gs >= NSA && !__all_sync(0xffffffffu, nxt_ready)) mbar_wait(&a_empty[sa], ((gs / NSA) + 1) & 1);
#ifdef PA_TRACE
        gw += clock64() - c0;
#endif
        PA_TR6(trc && it == 2 && tid == 0, 500 + j);
        tc_fence_after();
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int jt = 2 * j + i;   // E tile
          const uint32_t base = tm + lane_off + 128u + (uint32_t)(sa * 128 + i * 64 + gq * 32);
          if (jt < 64) {
            const uint32_t xb = xw[(jt >> 1) * NGEN + xt];
            const uint32_t bc = __byte_perm(xb, 0, (jt & 1) ? 0x3232 : 0x1010);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t o[16];
#pragma unroll
              for (int q = 0; q < 16; ++q) o[q] = hmul2_f16(bc, vr[h * 16 + q]);
              tmem_st16(base + (uint32_t)(h * 16), o);
            }
          } else if (jt < NBT && (!kUpd || gq == 0)) {
            // score-sum tile E_G[c][b]: A_b = x_b * (dden | 1), scaled like u
            const uint32_t dh = pack_f16(dsc * pv, dsc * pv);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              uint32_t o[16];
#pragma unroll
              for (int q = 0; q < 16; ++q) o[q] = hmul2_f16(dh, xw[(h * 16 + q) * NGEN + xt]);
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
        if (l == 0) mbar_arrive(&a_full[sa]);
        PA_TR6(trc && it == 2 && tid == 0, 600 + j);
      }
    }
#ifdef PA_TRACE
    if (trc && l == 0) {
      g_trace6[(kUpd ? 0 : 1024) + 720 + w * 2] = gw;
      g_trace6[(kUpd ? 0 : 1024) + 721 + w * 2] = gp;
      g_trace6[(kUpd ? 0 : 1024) + 760 + w * 2] = gr;
      g_trace6[(kUpd ? 0 : 1024) + 761 + w * 2] = gm;
    }
#endif
  } else if (w >= W_EPI && w < W_EPI + 8) {
    // epilogue: read the accumulator, zero it and hand it back, then add the fp32
    // intra-chunk part and store the final bf16 gradient rows
    const int e = w - W_EPI, gq = e >> 2, qd = w & 3, row = qd * 32 + l;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
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
    for (int it = 0, ti = blockIdx.x; ti < ntiles; ++it, ti += gridDim.x) {
      const ZvTile t = zv_tile(ti, nI, nk, kbeg);
      const int ab = it & 1;
      const int rr = kUpd ? row : gq * 128 + row;
      const bool live = t.I * TOK + rr < g.c;
      const int tok = t.k * g.c + t.I * TOK + rr;
      const bool is_dv = kUpd && gq == 1;
      {
        // the next tile's epilogue operands go to L2 now (a tile ahead): from HBM under
        // this kernel's load each dependent round trip costs several thousand cycles
        const int tn = ti + (int)gridDim.x;
        if (tn < ntiles) {
          const ZvTile u = zv_tile(tn, nI, nk, kbeg);
          const int tokn = u.k * g.c + u.I * TOK + rr;
          if (u.I * TOK + rr < g.c) {
            const char* o = (const char*)((is_dv ? dv32 : dx32) + ((size_t)u.s * g.t + tokn) * HD);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(o));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(o + 128));
            if (!is_dv) asm volatile("prefetch.global.L2 [%0];" ::"l"(xraw + rowid(g, u.s, tokn) * HD));
          }
        }
      }
      mbar_wait(&meta_full[ab], (it >> 1) & 1);
      const float fct = meta[ab * 256 + gq * 128 + row];
      __syncwarp();
      if (l == 0) mbar_arrive(&meta_empty[ab]);
      mbar_wait(acc_full, it & 1);
      PA_TR6(trc && it == 2 && tid == W_EPI * 32, 1);
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
      if (!live) continue;
      const size_t xr = rowid(g, t.s, tok);
      const float4* o32 = (const float4*)((is_dv ? dv32 : dx32) + ((size_t)t.s * g.t + tok) * HD);
      const uint4* xsrc = (const uint4*)(xraw + xr * HD);
      uint4* dst = (uint4*)((is_dv ? dvo : dxo) + xr * HD);
      float c = 0.f;
#pragma unroll
      for (int a4 = 0; a4 < 8; a4 += 4) {
        float4 ov[8];
        uint4 xv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          ov[2 * i] = o32[2 * (a4 + i)];
          ov[2 * i + 1] = o32[2 * (a4 + i) + 1];
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
            }
          }
          const float4 v0 = ov[2 * i], v1 = ov[2 * i + 1];
          dst[a] = make_uint4(pack_bf16(fmaf(f[0], fct, v0.x), fmaf(f[1], fct, v0.y)),
                              pack_bf16(fmaf(f[2], fct, v0.z), fmaf(f[3], fct, v0.w)),
                              pack_bf16(fmaf(f[4], fct, v1.x), fmaf(f[5], fct, v1.y)),
                              pack_bf16(fmaf(f[6], fct, v1.z), fmaf(f[7], fct, v1.w)));
        }
      }
      // d<., .>/d(log factor) = <dx~, x~>/2 (degree-2 homogeneity of phi')
      c *= 0.5f * fct;
      if (g.gated) {
        if (!kUpd) dell[(size_t)t.s * g.t + tok] += c;            // gp_m = exp(ell_m)
        else if (gq == 0) dellend[(size_t)t.s * g.t + tok] = c;   // suffix decay, finished in gate_finish
      }
      PA_TR6(trc && it == 2 && tid == W_EPI * 32, 2);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (w == W_TMA) tmem_dealloc<512>(tm);
}

// chunk 0 without a prefix has no state query: dq is the intra-chunk part alone
__global__ void __launch_bounds__(256) k_tc_dq_chunk0(Geo g, const float* __restrict__ dx32, __nv_bfloat16* dxo) {
  const int s = blockIdx.y;
  for (int i = blockIdx.x * 256 + threadIdx.x; i < g.c * 16; i += gridDim.x * 256) {
    const int r = i >> 4, c4 = (i & 15) * 4;
    const float4 v = *(const float4*)(dx32 + ((size_t)s * g.t + r) * HD + c4);
    *(uint2*)(dxo + rowid(g, s, r) * HD + c4) = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  }
}

int tc_zvjp(const Geo& g, bool upd, const CUtensorMap& m_x, const CUtensorMap& m_u, int u_bf16_bth,
            const __half* u16, const void* xraw, const float* ell, const float* lamlog, const __half* E,
            const float* dx32, const float* dv32, float* dell, float* dellend, void* dxo, void* dvo,
            cudaStream_t st) {
  using namespace zv;
  const int den = g.normalize ? 1 : 0;
  auto fn = upd ? (den ? k_tc_zvjp<true, 1> : k_tc_zvjp<true, 0>)
                : (den ? k_tc_zvjp<false, 1> : k_tc_zvjp<false, 0>);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int tok = upd ? 128 : 256;
  const int kbeg = (!upd && !g.prefix) ? 1 : 0;
  const int nI = (g.c + tok - 1) / tok, nk = g.n - kbeg;
  if (kbeg) {
    k_tc_dq_chunk0<<<dim3(8, g.ns), 256, 0, st>>>(g, dx32, (__nv_bfloat16*)dxo);
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
  fn<<<grid, THREADS, SMEM, st>>>(m_x, m_u, g, u_bf16_bth, u16, (const __nv_bfloat16*)xraw, ell, lamlog, E, dx32,
                                  dv32, dell, dellend, (__nv_bfloat16*)dxo, (__nv_bfloat16*)dvo, ntiles, nI, nk,
                                  kbeg);
  return 0;
}

}  // namespace pa
