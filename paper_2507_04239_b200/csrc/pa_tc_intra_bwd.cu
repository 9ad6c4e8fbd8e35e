// Intra-chunk backward in one pass (reference gradients.py:98-176, power
// branch, with the pairwise-decay chain rule 79-95 in log space): every
// causal 128 x 128 block pair of a chunk is visited once and feeds all three
// gradients -- five GEMMs per block pair, where a key-side and a query-side
// kernel that each recompute S and dP need seven.
//
// Per chunk with s = q.k (raw), E_ij = exp(ell_i - ell_j) for j <= i:
//   P = sigma^2 E s^2           dP' = dnum_i . v_j (+ dden_i, normalized)
//   T = sigma^2 E s              dS  = dP' T   (dq, dk carry a factor 2)
//   dV_J += P^T dnum_I     dK_J += dS^T Q_I     dQ_I += dS K_J
// Log-gate cotangents (gradients.py:79-95): dell_i += sum_j dP'_ij P_ij at the
// query, dell_j -= sum_i dP'_ij P_ij at the key, from the fp32 products.
//
// B200 design.  Persistent, one CTA per SM; a work item is (stream, chunk, key
// block pair J, nq-1-J), so every item holds nq + 1 block pairs (balanced).
// The key-major orientation keeps K_J / V_J resident (double-buffered) while
// 64-query half-blocks of Q and dnum stream through a 3-stage TMA ring:
//   issuer A (w21):  S^T = K_J Q_h^T, dP^T = V_J dnum_h^T  into one of two TMEM
//                    buffers (N = 64 each)
//   compute (w0-15): P^T, dS^T in bf16 written back in place (the A operand of
//                    the next GEMMs) and dS^T into a shared-memory tile
//   issuer B (w22):  dV_J += P^T dnum_h, dK_J += dS^T Q_h (TMEM A operand), and
//                    per query block dQ_I = dS K_J (dS MN-major from shared
//                    memory, M = 128 queries) into one of two dQ accumulators
//   epilogue (w16-19): dQ_I tiles are reduce-added to the fp32 dq buffer by TMA
//                    (cp.reduce.async.bulk); at the end of a key block dK_J,
//                    dV_J go out as bf16 rows by TMA store
//   w20: TMA loads and the TMEM allocation.
// Each accumulator is fed by one issuer in program order.  The dQ reduce-adds
// of different CTAs land in a timing-dependent order (deterministic mode runs
// the query side as its own pass instead, pa_tc_ib.cu).
#include <cuda.h>

#include "pa_common.cuh"
#include "pa_sm100.cuh"
#include "pa_tc.cuh"
#include "pa_tc_common.cuh"

namespace pa {
using namespace sm100;
using namespace tc;

#ifdef PA_TRACE
// debug build only (tools/trace_ix.py): clock64 stamps of one CTA, [event][index]
__device__ long long g_trace_ix[16 * 64];
extern "C" int pa_debug_trace_ix(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trace_ix, sizeof(long long) * n);
}
#define IX_TR(ev, i) \
  if (blockIdx.x == 7 && (i) < 64) g_trace_ix[(ev) * 64 + (i)] = clock64()
#else
#define IX_TR(ev, i)
#endif

namespace ibx {
constexpr int KV_B = 128 * 128;    // K_J or V_J: 128 tokens x 64 bf16 (SW128)
constexpr int H_B = 64 * 128;      // Q_h or dnum_h: 64 tokens x 64 bf16
constexpr int NQD = 3;             // half-block stages
constexpr int DS_B = 2 * 128 * 128;   // dS tile: 2 M-blocks (64 queries each) x 128 keys x 128 B (hi, then lo)
constexpr int STG_B = 32768;       // epilogue staging: dQ fp32 128 x 64, or dK + dV bf16
constexpr int OFF_KV = 0;
constexpr int OFF_QD = OFF_KV + 2 * 2 * KV_B;
constexpr int OFF_DS = OFF_QD + NQD * 2 * H_B;
constexpr int OFF_STG = OFF_DS + 2 * DS_B;   // one query block's dS hi and lo tiles
constexpr int OFF_F = OFF_STG + STG_B;     // ell, colf, rinv, cold: 4 x 1024 floats
constexpr int OFF_RED = OFF_F + 4 * 4096;  // key-side row sums [128]
constexpr int OFF_BAR = OFF_RED + 512;
// no static shared memory: the dynamic window starts 1024-aligned, so only a
// small slack is reserved (checked at run time) -- the budget is at the limit
constexpr int SMEM_PAD = 128;
constexpr int SMEM = SMEM_PAD + OFF_BAR + 256;
constexpr int NCW = 8;             // compute warps: two per SM sub-partition
constexpr int PPW = 16 / NCW;      // 16-column pieces per compute warp and half-block
constexpr int THREADS = 32 * (NCW + 7);   // + 4 epilogue, TMA + TMEM, issuer A, issuer B
constexpr int W_EPI = NCW, W_TMA = NCW + 4, W_MA = NCW + 5, W_MB = NCW + 6;
}  // namespace ibx

struct IbItem {
  int s, k, jp;
};
__device__ __forceinline__ IbItem ib_item(int it, int npair, int n) {
  IbItem r;
  r.jp = it % npair;
  const int rest = it / npair;
  r.k = rest % n;
  r.s = rest / n;
  return r;
}

__device__ __forceinline__ float ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

template <bool kNorm, bool kDQ>
__global__ void __launch_bounds__(ibx::THREADS, 1)
    k_tc_intra_bwd(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_dy,
                   const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dk,
                   const __grid_constant__ CUtensorMap tm_dv, Geo g, const float* __restrict__ ell,
                   const float* __restrict__ dden, const float* __restrict__ rsum,
                   const __nv_bfloat16* __restrict__ kraw, float* dell, int nitems) {
  using namespace ibx;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  if (pad > (uint32_t)SMEM_PAD) __trap();
  uint8_t* smem = smem_raw + pad;
  float* kred = (float*)(smem + OFF_RED);   // [128] key-side row sums over the column groups
  float* ell_s = (float*)(smem + OFF_F);   // in-chunk log2 prefix
  float* colf = ell_s + 1024;              // off-diagonal query factor sigma^2 2^(ell_i - ell_refJ) (/ R_i)
  float* rinv = colf + 1024;               // 1 / R_i (normalize)
  float* cold = rinv + 1024;               // dden_i R_i (normalize)
  uint64_t* bars = (uint64_t*)(smem + OFF_BAR);
  uint64_t* kv_full = bars;          // 2
  uint64_t* kv_empty = bars + 2;     // 2: issuers A and B
  uint64_t* qd_full = bars + 4;      // 3
  uint64_t* qd_empty = bars + 7;     // 3: issuers A and B
  uint64_t* s_full = bars + 10;      // 2
  uint64_t* p_full = bars + 12;      // 2: 8 compute warps
  uint64_t* sdp_free = bars + 14;    // 2
  uint64_t* dsm_free = bars + 16;    // 1: the dQ GEMM is done with the dS tiles
  uint64_t* ds_full = bars + 17;     // 1: a query block's dS tiles are written (compute warps)
  uint64_t* dq_full = bars + 18;     // 2
  uint64_t* dq_empty = bars + 20;    // 2: 4 epilogue warps
  uint64_t* acc_full = bars + 22;    // 1
  uint64_t* acc_empty = bars + 23;   // 1: 4 epilogue warps
  uint32_t* tmem_slot = (uint32_t*)(bars + 24);

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int nq = g.c / 128, npair = (nq + 1) / 2;
  const float sig2 = g.scale * g.scale;
  constexpr float LOG2E = 1.4426950408889634f;

  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 1);
      mbar_init(&kv_empty[i], 2);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], NCW);
      mbar_init(&sdp_free[i], 1);
      mbar_init(&dq_full[i], 1);
      mbar_init(&dq_empty[i], 4);
    }
    for (int i = 0; i < NQD; ++i) {
      mbar_init(&qd_full[i], 1);
      mbar_init(&qd_empty[i], 2);
    }
    mbar_init(acc_full, 1);
    mbar_init(acc_empty, 4);
    mbar_init(dsm_free, 1);
    mbar_init(ds_full, NCW);
    fence_barrier_init();
  }
  if (w == W_TMA) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tmem_slot;
  // TMEM: S/dP buffers b at [128 b, 128 b + 128) (S^T then dP^T, 64 columns each),
  // dV [256, 320), dK [320, 384), dQ buffers [384 + 64 x, ...)
  const uint32_t tDV = tm + 256, tDK = tm + 320;

  // the J list of an item: jp, then nq-1-jp when different
  auto njs = [&](int jp) { return (nq - 1 - jp != jp) ? 2 : 1; };
  auto jof = [&](int jp, int u) { return u == 0 ? jp : nq - 1 - jp; };

  if (w == W_TMA) {
    // one tensor per lane per copy, half-blocks alternating between two lane
    // pairs: a thread completes about one copy per 610 cycles whatever its size
    // (profiles/r01_tma_rate_probe.txt), about one half-block period
    if (l < 6) {
      if (l == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_dy);
      }
      int jn = 0, hn = 0;
      for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
        const IbItem wi = ib_item(it, npair, g.n);
        const int bi = wi.s / g.h, hi = wi.s % g.h, c0 = wi.k * g.c;
        for (int u = 0; u < njs(wi.jp); ++u, ++jn) {
          const int J = jof(wi.jp, u), jb = jn & 1;
          uint8_t* kv = smem + OFF_KV + jb * 2 * KV_B;
          if (l >= 4) {
            if (jn >= 2) mbar_wait(&kv_empty[jb], ((jn >> 1) + 1) & 1);
            if (l == 4) mbar_expect_tx(&kv_full[jb], 2 * KV_B);
            __syncwarp(0x30u);
            if (l == 4) tma_load_4d(kv, &tm_k, &kv_full[jb], 0, hi, c0 + J * 128, bi);
            if (l == 5) tma_load_4d(kv + KV_B, &tm_v, &kv_full[jb], 0, hi, c0 + J * 128, bi);
          }
          for (int I = J; I < nq; ++I)
            for (int h = 0; h < 2; ++h, ++hn) {
              if (l >= 4 || (l >> 1) != (hn & 1)) continue;
              const int st = hn % NQD;
              uint8_t* qd = smem + OFF_QD + st * 2 * H_B;
              if (hn >= NQD) mbar_wait(&qd_empty[st], ((hn / NQD) + 1) & 1);
              const unsigned pm = 3u << (2 * (hn & 1));
              if (!(l & 1)) mbar_expect_tx(&qd_full[st], 2 * H_B);
              __syncwarp(pm);
              const int tok = c0 + I * 128 + h * 64;
              if (!(l & 1)) tma_load_4d(qd, &tm_q, &qd_full[st], 0, hi, tok, bi);
              else tma_load_4d(qd + H_B, &tm_dy, &qd_full[st], 0, hi, tok, bi);
            }
        }
      }
    }
  } else if (w == W_MA) {
    // ---------------- issuer A: S^T and dP^T per half-block ----------------
    constexpr uint32_t idS = idesc_bf16(128, 64, false, false);
    int jn = 0, hn = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const IbItem wi = ib_item(it, npair, g.n);
      for (int u = 0; u < njs(wi.jp); ++u, ++jn) {
        const int J = jof(wi.jp, u), jb = jn & 1;
        mbar_wait_w(&kv_full[jb], (jn >> 1) & 1);
        // descriptor bases (K-major SW128); K-steps add 32 B = 2 units, V / dnum follow
        const uint64_t dK0 = smem_desc(smem_u32(smem + OFF_KV + jb * 2 * KV_B), 16, 1024, 2);
        for (int I = J; I < nq; ++I)
          for (int h = 0; h < 2; ++h, ++hn) {
            const int st = hn % NQD, b = hn & 1;
            mbar_wait_w(&qd_full[st], (hn / NQD) & 1);
            if (hn >= 2) mbar_wait_w(&sdp_free[b], ((hn >> 1) + 1) & 1);
            if (l == 0) IX_TR(0, hn);
            tc_fence_after();
            const uint64_t dQ0 = smem_desc(smem_u32(smem + OFF_QD + st * 2 * H_B), 16, 1024, 2);
            const uint32_t tS = tm + (uint32_t)(b * 128), tDP = tS + 64;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ss_w(tS, dK0 + (uint64_t)(kk * 2), dQ0 + (uint64_t)(kk * 2), idS, kk > 0 ? 1u : 0u);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              mma_ss_w(tDP, dK0 + (uint64_t)(KV_B >> 4) + (uint64_t)(kk * 2), dQ0 + (uint64_t)(H_B >> 4) + (uint64_t)(kk * 2),
                       idS, kk > 0 ? 1u : 0u);
            tc_commit_w(&s_full[b]);
            tc_commit_w(&qd_empty[st]);
            if (l == 0) IX_TR(1, hn);
          }
        tc_commit_w(&kv_empty[jb]);
      }
    }
  } else if (w == W_MB) {
    // ---------------- issuer B: dV, dK per half-block; dQ per query block ----------------
    constexpr uint32_t idG = idesc_bf16(128, 64, false, true);   // A TMEM, B MN-major
    constexpr uint32_t idQ = idesc_bf16(128, 64, true, true);    // A (dS) MN-major smem, B MN-major
    int jn = 0, hn = 0, In = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const IbItem wi = ib_item(it, npair, g.n);
      for (int u = 0; u < njs(wi.jp); ++u, ++jn) {
        const int J = jof(wi.jp, u), jb = jn & 1;
        mbar_wait_w(&kv_full[jb], (jn >> 1) & 1);
        // MN-major descriptor bases: K-steps of 16 rows add 2048 B = 128 units
        const uint64_t dKm = smem_desc(smem_u32(smem + OFF_KV + jb * 2 * KV_B), 8192, 1024, 2);
        const uint64_t dS0 = smem_desc(smem_u32(smem + OFF_DS), 16384, 1024, 2);
        bool first = true;
        for (int I = J; I < nq; ++I, ++In) {
          const int x = In & 1;
          for (int h = 0; h < 2; ++h, ++hn) {
            const int st = hn % NQD, b = hn & 1;
            mbar_wait_w(&p_full[b], (hn >> 1) & 1);
            if (l == 0) IX_TR(6, hn);
            if (first && jn >= 1) mbar_wait_w(acc_empty, (jn + 1) & 1);
            tc_fence_after();
            const uint64_t dQm = smem_desc(smem_u32(smem + OFF_QD + st * 2 * H_B), 8192, 1024, 2);
            const uint32_t tS = tm + (uint32_t)(b * 128), tDP = tS + 64;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
              const uint32_t acc = (first && kk == 0) ? 0u : 1u;
              // K-step kk: compute warp group kk / PPW, piece kk % PPW (in-place bf16)
              const uint32_t pc = (uint32_t)((kk / PPW) * 16 * PPW + (kk % PPW) * 8);
              mma_ts_w(tDV, tS + pc, dQm + (uint64_t)(H_B >> 4) + (uint64_t)(kk * 128), idG, acc);
              mma_ts_w(tDK, tDP + pc, dQm + (uint64_t)(kk * 128), idG, acc);
            }
            first = false;
            tc_commit_w(&sdp_free[b]);
            tc_commit_w(&qd_empty[st]);
            if (l == 0) IX_TR(7, hn);
          }
          if (kDQ) {
            if (In >= 2) mbar_wait_w(&dq_empty[x], ((In >> 1) + 1) & 1);
            mbar_wait_w(ds_full, In & 1);
            IX_TR(8, In);
            tc_fence_after();
            const uint32_t tDQ = tm + 384u + (uint32_t)(x * 64);
            // dQ_I = (dS_hi + dS_lo) K_J: the fp32 dq rows then carry dS to ~2^-17, so
            // <q, dq>/2 matches the key side's fp32 sum_i dS s pair by pair
#pragma unroll
            for (int kk = 0; kk < 16; ++kk)
              mma_ss_w(tDQ, dS0 + (uint64_t)((kk >> 3) * (DS_B >> 4) + (kk & 7) * 128), dKm + (uint64_t)((kk & 7) * 128), idQ,
                       kk > 0 ? 1u : 0u);
            tc_commit_w(&dq_full[x]);
          }
          tc_commit_w(dsm_free);
        }
        tc_commit_w(acc_full);
        tc_commit_w(&kv_empty[jb]);
      }
    }
  } else if (w < NCW) {
    // ---------------- compute: P^T, dS^T ----------------
    // lane quadrant q (key rows 32 q .. 32 q + 31 of the block), column group cg
    // (16 PPW columns of each 64-query half-block) as PPW pieces of 16 columns
    const int q = w & 3, cg = w >> 2, row = q * 32 + l;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    if (tid < 128) kred[tid] = 0.f;
    // the per-item tables (ell, and R, dden when normalizing) are fetched into
    // registers one key block ahead, so an item switch does not wait on memory
    constexpr int NPF = 1024 / (NCW * 32);
    float pf_l[NPF], pf_r[NPF], pf_d[NPF];
    auto fetch = [&](const IbItem& f) {
#pragma unroll
      for (int r = 0; r < NPF; ++r) {
        const int i = tid + r * NCW * 32;
        if (i < g.c) {
          const int m = f.k * g.c + i;
          pf_l[r] = ell[(size_t)f.s * g.t + m];
          if (kNorm) {
            pf_r[r] = rsum[rowid(g, f.s, m)];
            pf_d[r] = dden[(size_t)f.s * g.t + m];
          }
        }
      }
    };
    int jn = 0, hn = 0, In = 0;
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const IbItem wi = ib_item(it, npair, g.n);
      const int c0 = wi.k * g.c;
      if (it == (int)blockIdx.x) fetch(wi);
      named_bar(1, NCW * 32);   // every compute warp is done with the previous item's tables
#pragma unroll
      for (int r = 0; r < NPF; ++r) {
        const int i = tid + r * NCW * 32;
        if (i < g.c) {
          ell_s[i] = LOG2E * pf_l[r];
          if (kNorm) {
            // rows past the caller's sequence (zero padding) have R = 0: weight 0
            rinv[i] = c0 + i < g.treal ? 1.f / pf_r[r] : 0.f;
            cold[i] = pf_d[r] * pf_r[r];
          }
        }
      }
      for (int u = 0; u < njs(wi.jp); ++u, ++jn) {
        const int J = jof(wi.jp, u);
        named_bar(1, NCW * 32);
        const float lref = ell_s[J * 128 + 127];
        for (int i = J * 128 + tid; i < g.c; i += NCW * 32) {
          float f = sig2 * ex2(fminf(ell_s[i] - lref, 0.f));
          if (kNorm) f *= rinv[i];
          colf[i] = f;
        }
        named_bar(1, NCW * 32);
        if (u == njs(wi.jp) - 1 && it + (int)gridDim.x < nitems) fetch(ib_item(it + gridDim.x, npair, g.n));
        const int key = J * 128 + row;             // chunk-relative key of this TMEM lane
        const float l_key = ell_s[key];
        const float rowf = ex2(fminf(lref - l_key, 0.f));
        const f2v rowf2 = {rowf, rowf};
        // key-side log-gate cotangent sum_i dP' P = sum_i dS s (fp32, unrounded)
        f2v red = {0.f, 0.f};
        for (int I = J; I < nq; ++I, ++In) {
          const bool diag = I == J;
          for (int h = 0; h < 2; ++h, ++hn) {
            const int b = hn & 1;
            mbar_wait(&s_full[b], (hn >> 1) & 1);
            if (tid == 0) IX_TR(2, hn);
            tc_fence_after();
            const uint32_t tS = tm + (uint32_t)(b * 128), tDP = tS + 64;
            // phase 1 (critical path of the dV / dK GEMMs): P^T, dS^T in bf16 back
            // into TMEM; phase 2 after the arrival: the dS hi / lo tiles for the dQ GEMM
            float dsv[PPW][16];
            uint32_t pdk[PPW][8];
#pragma unroll
            for (int pc = 0; pc < PPW; ++pc) {
              const int cofs = (cg * PPW + pc) * 16;             // column inside the half-block
              const int qb = I * 128 + h * 64 + cofs;            // chunk-relative query of the first column
              uint32_t rs[16], rd[16], pp[8];
              uint32_t* pd = pdk[pc];
              tmem_ld16(tS + lane_off + cofs, rs);
              tmem_ld16(tDP + lane_off + cofs, rd);
              tc_wait_ld();
              if (!diag) {
#pragma unroll
                for (int e4 = 0; e4 < 4; ++e4) {
                  const float4 cf = *(const float4*)(colf + qb + e4 * 4);
                  float4 cd = make_float4(0.f, 0.f, 0.f, 0.f);
                  if (kNorm) cd = *(const float4*)(cold + qb + e4 * 4);
#pragma unroll
                  for (int z = 0; z < 2; ++z) {
                    const int e = e4 * 4 + z * 2;
                    const f2v sv = {__uint_as_float(rs[e]), __uint_as_float(rs[e + 1])};
                    f2v dp = {__uint_as_float(rd[e]), __uint_as_float(rd[e + 1])};
                    if (kNorm) dp = add2v(dp, z ? f2v{cd.z, cd.w} : f2v{cd.x, cd.y});
                    const f2v T = mul2v(mul2v(z ? f2v{cf.z, cf.w} : f2v{cf.x, cf.y}, rowf2), sv);
                    const f2v P = mul2v(T, sv);
                    const f2v dS = mul2v(dp, T);
                    pp[e >> 1] = pack_bf16(P.x, P.y);
                    pd[e >> 1] = pack_bf16(dS.x, dS.y);
                    dsv[pc][e] = dS.x;
                    dsv[pc][e + 1] = dS.y;
                    red = fma2v(dS, sv, red);
                  }
                }
              } else if (qb + 15 < key) {
#pragma unroll
                for (int e = 0; e < 8; ++e) pp[e] = pd[e] = 0u;
#pragma unroll
                for (int e = 0; e < 16; ++e) dsv[pc][e] = 0.f;
              } else {
                // diagonal block: exact 2^(ell_i - ell_j) under the causal mask (query >= key)
#pragma unroll
                for (int e4 = 0; e4 < 4; ++e4) {
                  const float4 lc = *(const float4*)(ell_s + qb + e4 * 4);
                  float4 cd = make_float4(0.f, 0.f, 0.f, 0.f), ri = make_float4(1.f, 1.f, 1.f, 1.f);
                  if (kNorm) {
                    cd = *(const float4*)(cold + qb + e4 * 4);
                    ri = *(const float4*)(rinv + qb + e4 * 4);
                  }
                  const float lcv[4] = {lc.x, lc.y, lc.z, lc.w};
                  const float cdv[4] = {cd.x, cd.y, cd.z, cd.w};
                  const float riv[4] = {ri.x, ri.y, ri.z, ri.w};
                  float Pv[4];
#pragma unroll
                  for (int z = 0; z < 4; ++z) {
                    const int e = e4 * 4 + z;
                    const float sv = __uint_as_float(rs[e]);
                    float dp = __uint_as_float(rd[e]);
                    if (kNorm) dp += cdv[z];
                    float E = (qb + e >= key) ? sig2 * ex2(fminf(lcv[z] - l_key, 0.f)) : 0.f;
                    if (kNorm) E *= riv[z];
                    const float T = E * sv;
                    Pv[z] = T * sv;
                    dsv[pc][e] = dp * T;
                    red.x = fmaf(dsv[pc][e], sv, red.x);
                  }
                  pp[e4 * 2] = pack_bf16(Pv[0], Pv[1]);
                  pp[e4 * 2 + 1] = pack_bf16(Pv[2], Pv[3]);
                  pd[e4 * 2] = pack_bf16(dsv[pc][e4 * 4], dsv[pc][e4 * 4 + 1]);
                  pd[e4 * 2 + 1] = pack_bf16(dsv[pc][e4 * 4 + 2], dsv[pc][e4 * 4 + 3]);
                }
              }
              // in place: the bf16 pairs of this piece's 16 columns land in 8 u32
              // columns of this warp's own, already-read range (K-step cg PPW + pc of
              // the dV / dK GEMMs)
              const uint32_t pcl = (uint32_t)(cg * PPW * 16 + pc * 8);
              tmem_st8(tS + lane_off + pcl, pp);
              tmem_st8(tDP + lane_off + pcl, pd);
            }
            tc_wait_st();
            tc_fence_before();
            __syncwarp();
            if (tid == 0) IX_TR(3, hn);
            if (l == 0) mbar_arrive(&p_full[b]);
            if (kDQ) {
              // dS^T = hi + lo (bf16 each) for the dQ GEMM: row `row` into M-block h
              // of the two tiles (MN-major SW128: [128 keys][64 queries] bf16); the
              // previous query block's dQ GEMM must be done with them
              if (h == 0 && In >= 1) mbar_wait(dsm_free, (In - 1) & 1);
#pragma unroll
              for (int pc = 0; pc < PPW; ++pc) {
                const int cofs = (cg * PPW + pc) * 16;
                uint32_t pl[8];
#pragma unroll
                for (int e2 = 0; e2 < 8; ++e2) {
                  const float2 hi = __bfloat1622float2(*(const __nv_bfloat162*)&pdk[pc][e2]);
                  pl[e2] = pack_bf16(dsv[pc][2 * e2] - hi.x, dsv[pc][2 * e2 + 1] - hi.y);
                }
                uint8_t* rp = smem + OFF_DS + h * 16384 + row * 128;
                const int ch = cofs >> 3;
                const uint32_t o0 = (uint32_t)((ch ^ (row & 7)) << 4), o1 = (uint32_t)(((ch + 1) ^ (row & 7)) << 4);
                const uint32_t* pd = pdk[pc];
                *(uint4*)(rp + o0) = make_uint4(pd[0], pd[1], pd[2], pd[3]);
                *(uint4*)(rp + o1) = make_uint4(pd[4], pd[5], pd[6], pd[7]);
                *(uint4*)(rp + DS_B + o0) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
                *(uint4*)(rp + DS_B + o1) = make_uint4(pl[4], pl[5], pl[6], pl[7]);
              }
              if (h == 1) {
                fence_async_smem();
                __syncwarp();
                if (l == 0) mbar_arrive(ds_full);
              }
            }
          }
        }
        if (g.gated) {
          // key side: dell_j -= sum_i dS_ij s_ij over the key block's queries
          // (the query side, + <q, dq>/2, is added from the fp32 dq rows by the
          // state-VJP kernel; both see the same dS to ~2^-17)
          atomicAdd(kred + row, red.x + red.y);
          named_bar(1, NCW * 32);
          if (cg == 0) {
            atomicAdd(dell + (size_t)wi.s * g.t + c0 + key, -kred[row]);
            kred[row] = 0.f;
          }
        }
      }
    }
  } else if (w >= W_EPI && w < W_EPI + 4) {
    // ---------------- epilogue: dQ reduce-adds, dK / dV stores ----------------
    const int q = w & 3, row = q * 32 + l, et = tid - W_EPI * 32;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    uint8_t* stg = smem + OFF_STG;
    int jn = 0, In = 0;
    auto staging_free = [&]() {
      if (et == 0) bulk_wait_read0();
      named_bar(2, 128);
    };
    for (int it = blockIdx.x; it < nitems; it += gridDim.x) {
      const IbItem wi = ib_item(it, npair, g.n);
      const int c0 = wi.k * g.c;
      for (int u = 0; u < njs(wi.jp); ++u, ++jn) {
        const int J = jof(wi.jp, u);
        for (int I = J; I < nq; ++I, ++In) {
          if (!kDQ) continue;
          const int x = In & 1;
          mbar_wait(&dq_full[x], (In >> 1) & 1);
          if (et == 0) IX_TR(9, In);
          tc_fence_after();
          const uint32_t tDQ = tm + 384u + (uint32_t)(x * 64) + lane_off;
          staging_free();
          // fp32 rows, factor 2 (dS carries 1/2), as two SW128 halves of 32 columns
#pragma unroll
          for (int hc = 0; hc < 2; ++hc) {
            uint32_t r[32];
            tmem_ld32(tDQ + hc * 32, r);
            tc_wait_ld();
            if (hc == 1) {
              tc_fence_before();
              __syncwarp();
              if (l == 0) mbar_arrive(&dq_empty[x]);
            }
#pragma unroll
            for (int c4 = 0; c4 < 8; ++c4) {
              const uint32_t* v = r + c4 * 4;
              *(float4*)(stg + hc * 16384 + row * 128 + ((c4 ^ (row & 7)) << 4)) =
                  make_float4(2.f * __uint_as_float(v[0]), 2.f * __uint_as_float(v[1]),
                              2.f * __uint_as_float(v[2]), 2.f * __uint_as_float(v[3]));
            }
          }
          fence_async_smem();
          named_bar(2, 128);
          if (et == 0) {
            const int r0 = wi.s * g.t + c0 + I * 128;
            tma_reduce_add_2d(&tm_dq, stg, 0, r0);
            tma_reduce_add_2d(&tm_dq, stg + 16384, 32, r0);
            bulk_commit();
            IX_TR(10, In);
          }
        }
        // key block J complete: dV (P' carries sigma^2) and dK (x 2) as bf16 rows,
        // one accumulator at a time (64 registers)
        mbar_wait(acc_full, jn & 1);
        tc_fence_after();
        staging_free();
#pragma unroll
        for (int which = 0; which < 2; ++which) {
          uint32_t a[64];
          const uint32_t src = (which ? tDK : tDV) + lane_off;
          const float f = which ? 2.f : 1.f;
          tmem_ld32(src, a);
          tmem_ld32(src + 32, a + 32);
          tc_wait_ld();
          if (which) {
            tc_fence_before();
            __syncwarp();
            if (l == 0) mbar_arrive(acc_empty);
          }
#pragma unroll
          for (int c8 = 0; c8 < 8; ++c8) {
            const uint32_t* v = a + c8 * 8;
            *(uint4*)(stg + which * 16384 + row * 128 + ((c8 ^ (row & 7)) << 4)) =
                make_uint4(pack_bf16(f * __uint_as_float(v[0]), f * __uint_as_float(v[1])),
                           pack_bf16(f * __uint_as_float(v[2]), f * __uint_as_float(v[3])),
                           pack_bf16(f * __uint_as_float(v[4]), f * __uint_as_float(v[5])),
                           pack_bf16(f * __uint_as_float(v[6]), f * __uint_as_float(v[7])));
          }
        }
        fence_async_smem();
        named_bar(2, 128);
        if (et == 0) {
          const int r0 = wi.s * g.t + c0 + J * 128;
          tma_store_2d(&tm_dv, stg, 0, r0);
          tma_store_2d(&tm_dk, stg + 16384, 0, r0);
          bulk_commit();
        }
      }
    }
    if (et == 0) bulk_wait0();
  }
  tc_fence_before();
  __syncthreads();
  if (w == W_TMA) tmem_dealloc<512>(tm);
}

int tc_intra_bwd_fused(const Geo& g, const void* q, const void* k, const void* v, const void* dy, const float* ell,
                       const float* dden, const float* rsum, __nv_bfloat16* dk16, __nv_bfloat16* dv16, float* dq32,
                       float* dell, cudaStream_t st) {
  using namespace ibx;
  CUtensorMap m_q, m_k, m_v, m_dy, m_dq, m_dk, m_dv;
  const size_t rows = (size_t)g.ns * g.t;
  if (!tc_map_bth(&m_q, q, g, 64) || !tc_map_bth(&m_k, k, g, 128) || !tc_map_bth(&m_v, v, g, 128) ||
      !tc_map_bth(&m_dy, dy, g, 64) || !tc_map_2d(&m_dq, dq32, rows, HD, 32, 128, 1) ||
      !tc_map_2d(&m_dk, dk16, rows, HD, 64, 128, 0) || !tc_map_2d(&m_dv, dv16, rows, HD, 64, 128, 0))
    return 3;
  const bool dq = !g.det;
  if (dq) cudaMemsetAsync(dq32, 0, rows * HD * sizeof(float), st);
  auto fn = g.normalize ? (dq ? k_tc_intra_bwd<true, true> : k_tc_intra_bwd<true, false>)
                        : (dq ? k_tc_intra_bwd<false, true> : k_tc_intra_bwd<false, false>);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int nitems = g.ns * g.n * ((g.c / 128 + 1) / 2);
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  fn<<<nitems < nsm ? nitems : nsm, THREADS, SMEM, st>>>(m_q, m_k, m_v, m_dy, m_dq, m_dk, m_dv, g, ell, dden, rsum,
                                                         (const __nv_bfloat16*)k, dell, nitems);
  count_launch();
  return 0;
}

}  // namespace pa
