// Intra-chunk backward on tcgen05 (reference gradients.py:98-176, power branch,
// with the pairwise-decay chain rule 79-95 taken in log space) -- the
// two-kernel form.  Only its query side is launched: in deterministic mode
// (PA_FLAG_DETERMINISTIC) it computes dQ with a fixed summation order, next to
// the one-pass kernel of pa_tc_intra_bwd.cu running without its dQ reduce-adds.
//
// Per chunk, with s = q.k (raw), E_ij = exp(ell_i - ell_j) for j <= i:
//   P = sigma^2 E s^2,   dP' = dnum.v + dden,   dS = 2 sigma^2 E dP' s
//   key side  (kKV):  dV_J = sum_I P^T dnum_I,  dK_J = sum_I dS^T Q_I,  dell_j -= sum_i dP' P
//   query side:       dQ_I = sum_J dS K_J,                            dell_i += sum_j dP' P
//
// Design (B200): two CTAs per SM (256 TMEM columns, ~110 KB shared memory,
// 384 threads each) so one CTA's elementwise phase overlaps the other's MMAs and the two
// CTAs' tcgen05 issue streams interleave (one CTA alone is capped at ~72% of
// the tensor peak by the per-CTA MMA issue interval at N = 64, see
// profiles/r01_mma_rate_probe.txt).  The streamed 128-token block is
// processed as two 64-token sub-blocks: S/dP for a sub-block use 128 TMEM
// columns, P and dS are written back in place as bf16 (the gradient MMAs read
// them as the TMEM A operand), and the two 64-column gradient accumulators
// take the other 128 columns.
// Off-diagonal blocks use the factorisation E_ij = r_i c_j with both factors
// <= 1 (referenced to the end of the key block); the diagonal block evaluates
// exp(ell_i - ell_j) per element under the causal mask.
#include <cuda.h>

#include "pa_common.cuh"
#include "pa_sm100.cuh"
#include "pa_tc.cuh"
#include "pa_tc_common.cuh"

namespace pa {
using namespace sm100;
using namespace tc;

#ifdef PA_TRACE
// debug build only (tools/trace_ib.py): clock64 stamps of one CTA's pipeline
__device__ long long g_trace[1024];
extern "C" int pa_debug_trace(long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(long long) * n);
}
#define PA_TR(i) \
  if (tr) g_trace[(i)] = clock64()
#else
#define PA_TR(i)
#endif

namespace ib2 {
constexpr int T128 = 128 * 128;   // one 128-token x 64 bf16 tile
constexpr int NST = 2;            // streamed-tile stages
// Warp roles: w0..w7 compute, w8 TMEM owner, w9 TMA, w10 MMA.  The issuing
// warps get the highest warp ids: the scheduler prefers high ids, so spinning
// compute warps cannot starve the MMA / TMA issue.
constexpr int THREADS = 352;
constexpr int W_TMEM = 8, W_TMA = 9, W_MMA = 10;
constexpr int SMEM = 1024 + 2 * T128 + NST * 2 * T128 + 3 * 4096 + 512 + 256;
}  // namespace ib2

struct f2 {
  float x, y;
};
__device__ __forceinline__ uint64_t u64(f2 a) { return *(uint64_t*)&a; }
__device__ __forceinline__ f2 mk(uint64_t r) { return *(f2*)&r; }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u64(a)), "l"(u64(b)));
  return mk(r);
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u64(a)), "l"(u64(b)));
  return mk(r);
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(u64(a)), "l"(u64(b)), "l"(u64(c)));
  return mk(r);
}

__device__ __forceinline__ float exp2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// TMEM column of the bf16 P / dS K-chunk kk (16 tokens): compute-warp group kk/2,
// piece kk%2 (see the in-place write in the compute warps)
__device__ __forceinline__ uint32_t pcol(int kk) { return (uint32_t)((kk >> 1) * 32 + (kk & 1) * 8); }

// kKV = true: one CTA per key block J, loops query blocks I = J..nq-1.
// kKV = false: one CTA per query block I (heaviest first), loops key blocks J = 0..I.
template <bool kKV, bool kNorm>
__global__ void __launch_bounds__(ib2::THREADS, 2) k_tc_ib(const __grid_constant__ CUtensorMap tm_q,
                                                  const __grid_constant__ CUtensorMap tm_k,
                                                  const __grid_constant__ CUtensorMap tm_v,
                                                  const __grid_constant__ CUtensorMap tm_dn, Geo g,
                                                  const float* __restrict__ ell, const float* __restrict__ dden,
                                                  const float* __restrict__ rsum, float* out_a, float* out_b,
                                                  float* dell) {
  using namespace ib2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* f0 = smem;                      // kKV: K_J   | q-side: Q_I
  uint8_t* f1 = f0 + T128;                 // kKV: V_J   | q-side: dN_I
  uint8_t* s0 = f1 + T128;                 // stages: kKV: (Q_X, dN_X) | q-side: (K_X, V_X)
  float* ell_s = (float*)(s0 + NST * 2 * T128);   // [1024] in-chunk log prefix
  float* colf = ell_s + 1024;                       // [1024] off-diagonal column factor
  float* cold = colf + 1024;                        // [1024] dden per query column (kKV, normalize)
  float* cinv = cold + 1024;                        // [128] 1/rowsum of the diagonal block's query columns
  uint64_t* bars = (uint64_t*)(cinv + 128);
  uint64_t* f_full = bars;
  uint64_t* t_full = f_full + 1;         // NST
  uint64_t* t_empty = t_full + NST;      // NST
  uint64_t* s_full = t_empty + NST;      // S / dP of the current sub-block in TMEM
  uint64_t* p_full = s_full + 1;         // P / dS written back (4 compute warps)
  uint64_t* fin = p_full + 1;
  __shared__ uint32_t tmem_base;

  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31;
  const int nq = g.c / 128;
  const int B0 = kKV ? (int)blockIdx.x : nq - 1 - (int)blockIdx.x;
  const int k = blockIdx.y, s = blockIdx.z;
  const int bi = s / g.h, hi = s % g.h;
  const int c0 = k * g.c;
  const int nblk = kKV ? nq - B0 : B0 + 1;
  const float sig2 = g.scale * g.scale;
#ifdef PA_TRACE
  const bool tr0 = kKV && blockIdx.x == 0 && blockIdx.y == 5 && blockIdx.z == 3;
#endif

  if (w == W_TMEM) tmem_alloc<256>(&tmem_base);
  if (tid == 0) {
    mbar_init(f_full, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 8);
    mbar_init(fin, 1);
    fence_barrier_init();
  }
  constexpr float LOG2E = 1.4426950408889634f;
  for (int i = tid; i < g.c; i += THREADS) ell_s[i] = LOG2E * ell[(size_t)s * g.t + c0 + i];
  __syncthreads();
  // column factors (both <= 1): kKV  r_i = sigma^2 exp(ell_i - ell_endJ)   (queries after block J)
  //                             q-side c_j = exp(ell_end(J(j)) - ell_j)    (keys, own block end)
  {
    const float lrefJ = ell_s[B0 * 128 + 127];
    const int lim = kKV ? g.c : (B0 + 1) * 128;
    for (int i = tid; i < lim; i += THREADS) {
      if (kKV)
        colf[i] = sig2 * exp2_approx(fminf(ell_s[i] - lrefJ, 0.f));
      else
        colf[i] = exp2_approx(fminf(ell_s[(i | 127)] - ell_s[i], 0.f));
      if (kKV && kNorm) {
        // normalization (gradients.py:381-386) with the 1/rowsum folded into the
        // column factor: the dP GEMM runs on the exact bf16 dy, and
        //   dP' = (dy.v - dy.y) / R = (acc + dden R) / R
        // so with c' = c / R: P' = P / R (the dV operand, = P^T dnum), dS = (acc + dden R) T'
        const float R = rsum[rowid(g, s, c0 + i)];
        const float Ri = c0 + i < g.treal ? 1.f / R : 0.f;   // zero padding past the sequence: weight 0
        colf[i] *= Ri;
        cold[i] = dden[(size_t)s * g.t + c0 + i] * R;
        if ((i >> 7) == B0) cinv[i & 127] = Ri;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tmem_base;
  const uint32_t tS = tm, tDP = tm + 64, tA = tm + 128, tB = tm + 192;

  if (w == W_TMA) {
    // dy rows ([b, t, h, 64]); normalization is applied in fp32 (see cold / rinv_own)
    auto load_dn = [&](void* dst, uint64_t* bar, int blk) { tma_load_4d(dst, &tm_dn, bar, 0, hi, c0 + blk * 128, bi); };
    // two issuing lanes (one per tensor): a thread completes one TMA copy per ~610
    // cycles whatever its size (profiles/r01_bulk_copy_probe.txt)
    if (l < 2) {
      if (l == 0) {
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
        tma_prefetch(&tm_dn);
        mbar_expect_tx(f_full, 2 * T128);
      }
      __syncwarp(3u);
      if (kKV) {
        if (l == 0) tma_load_4d(f0, &tm_k, f_full, 0, hi, c0 + B0 * 128, bi);
        if (l == 1) tma_load_4d(f1, &tm_v, f_full, 0, hi, c0 + B0 * 128, bi);
      } else {
        if (l == 0) tma_load_4d(f0, &tm_q, f_full, 0, hi, c0 + B0 * 128, bi);
        if (l == 1) load_dn(f1, f_full, B0);
      }
      for (int it = 0; it < nblk; ++it) {
        const int X = kKV ? B0 + it : it, st = it % NST;
        if (it >= NST) mbar_wait(&t_empty[st], ((it / NST) + 1) & 1);
        if (l == 0) mbar_expect_tx(&t_full[st], 2 * T128);
        __syncwarp(3u);
        uint8_t* d0 = s0 + st * 2 * T128;
        if (kKV) {
          if (l == 0) tma_load_4d(d0, &tm_q, &t_full[st], 0, hi, c0 + X * 128, bi);
          if (l == 1) load_dn(d0 + T128, &t_full[st], X);
        } else {
          if (l == 0) tma_load_4d(d0, &tm_k, &t_full[st], 0, hi, c0 + X * 128, bi);
          if (l == 1) tma_load_4d(d0 + T128, &tm_v, &t_full[st], 0, hi, c0 + X * 128, bi);
        }
      }
    }
  } else if (w == W_MMA) {
    {
      constexpr uint32_t idS = idesc_bf16(128, 64, false, false);   // S / dP: both K-major
      constexpr uint32_t idG = idesc_bf16(128, 64, false, true);    // gradients: B MN-major
      mbar_wait_w(f_full, 0);
      const uint32_t F0 = smem_u32(f0), F1 = smem_u32(f1);
      for (int it = 0; it < nblk; ++it) {
        const int st = it % NST;
        mbar_wait_w(&t_full[st], (it / NST) & 1);
        tc_fence_after();
        const uint32_t T0 = smem_u32(s0 + st * 2 * T128), T1 = T0 + T128;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int n = it * 2 + h;
#ifdef PA_TRACE
          const bool tr = tr0 && n < 64;
#endif
          PA_TR(n * 8 + 0);
          const uint32_t hb = (uint32_t)h * 8192u;   // 64 rows x 128 B
          // kKV: S^T = K_J Q_h^T, dP^T = V_J dN_h^T   | q-side: S = Q_I K_h^T, dP = dN_I V_h^T
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            mma_ss_w(tS, smem_desc(F0 + kk * 32, 16, 1024, 2), smem_desc(T0 + hb + kk * 32, 16, 1024, 2), idS,
                   kk > 0 ? 1u : 0u);
            mma_ss_w(tDP, smem_desc(F1 + kk * 32, 16, 1024, 2), smem_desc(T1 + hb + kk * 32, 16, 1024, 2), idS,
                   kk > 0 ? 1u : 0u);
          }
          tc_commit_w(s_full);
          PA_TR(n * 8 + 1);
          mbar_wait_w(p_full, n & 1);
          PA_TR(n * 8 + 2);
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t acc = (n > 0 || kk > 0) ? 1u : 0u;
            if (kKV) {
              mma_ts_w(tA, tS + pcol(kk), smem_desc(T1 + hb + kk * 2048, 8192, 1024, 2), idG, acc);   // dV += P^T dN
              mma_ts_w(tB, tDP + pcol(kk), smem_desc(T0 + hb + kk * 2048, 8192, 1024, 2), idG, acc);  // dK += dS^T Q
            } else {
              mma_ts_w(tA, tDP + pcol(kk), smem_desc(T0 + hb + kk * 2048, 8192, 1024, 2), idG, acc);  // dQ += dS K
            }
          }
          PA_TR(n * 8 + 3);
        }
        tc_commit_w(&t_empty[st]);
      }
      tc_commit_w(fin);
    }
  } else if (w < 8) {
    // 8 compute warps: lane quadrant q = w % 4, column half grp = w / 4 of
    // each 64-column sub-block, processed as two 16-column pieces.
    const int q = w & 3, grp = w >> 2, row = q * 32 + l;
    const uint32_t lane_off = (uint32_t)(q * 32) << 16;
    const int own = B0 * 128 + row;            // chunk-relative token of this TMEM lane
    const float l_own = ell_s[own];            // log2 units
    // q-side normalization: the row factor takes 1/R_own, dden takes R_own (see cold above)
    const float R_own = (!kKV && kNorm) ? rsum[rowid(g, s, c0 + own)] : 1.f;
    const float dden_own = (!kKV && kNorm) ? dden[(size_t)s * g.t + c0 + own] * R_own : 0.f;
    const float rinv_own = c0 + own < g.treal ? 1.f / R_own : 0.f;   // zero padding: weight 0
    // kKV: c_own = 2^(ell_endJ - ell_own) (<= 1); q-side: r_own = sigma^2 2^(ell_own - ell_endJ) per J
    const float c_own = kKV ? exp2_approx(fminf(ell_s[B0 * 128 + 127] - l_own, 0.f)) : 0.f;
    f2 red = {0.f, 0.f};
    for (int n = 0; n < 2 * nblk; ++n) {
      const int it = n >> 1, h = n & 1;
      const int X = kKV ? B0 + it : it;
      const bool diag = (X == B0);
      const float rowf =
          kKV ? c_own : sig2 * exp2_approx(fminf(l_own - ell_s[X * 128 + 127], 0.f)) * rinv_own;
      const f2 rowf2 = {rowf, rowf};
#ifdef PA_TRACE
      const bool tr = tr0 && n < 64 && w == 0 && l == 0;
#endif
      PA_TR(n * 8 + 4);
      mbar_wait(s_full, n & 1);
      PA_TR(n * 8 + 5);
      tc_fence_after();
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int cofs = grp * 32 + hh * 16;              // column offset inside the sub-block
        const int colbase = X * 128 + h * 64 + cofs;      // chunk-relative token of the first column
        uint32_t rs[16], rd[16], pp[8], pd[8];
        tmem_ld16(tS + lane_off + cofs, rs);
        tmem_ld16(tDP + lane_off + cofs, rd);
        tc_wait_ld();
        // the causal mask of the diagonal block: kKV needs col >= own, q-side col <= own
        const bool all_masked = diag && (kKV ? (colbase + 15 < own) : (colbase > own));
        if (!diag) {
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const float4 cf = *(const float4*)(colf + colbase + e4 * 4);
            float4 cd = make_float4(0.f, 0.f, 0.f, 0.f);
            if (kKV && kNorm) cd = *(const float4*)(cold + colbase + e4 * 4);
#pragma unroll
            for (int z = 0; z < 2; ++z) {
              const int e = e4 * 4 + z * 2;
              const f2 sv = {__uint_as_float(rs[e]), __uint_as_float(rs[e + 1])};
              f2 dp = {__uint_as_float(rd[e]), __uint_as_float(rd[e + 1])};
              const f2 cc = z ? f2{cf.z, cf.w} : f2{cf.x, cf.y};
              if (kNorm) dp = add2(dp, kKV ? (z ? f2{cd.z, cd.w} : f2{cd.x, cd.y}) : f2{dden_own, dden_own});
              const f2 T = mul2(mul2(cc, rowf2), sv);
              const f2 P = mul2(T, sv);
              const f2 dS = mul2(dp, T);
              red = fma2(dp, P, red);
              pp[e >> 1] = pack_bf16(P.x, P.y);
              pd[e >> 1] = pack_bf16(dS.x, dS.y);
            }
          }
        } else if (all_masked) {
#pragma unroll
          for (int e = 0; e < 8; ++e) pp[e] = pd[e] = 0u;
        } else {
          // diagonal block: exact 2^(ell_i - ell_j) under the causal mask
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const float4 lc = *(const float4*)(ell_s + colbase + e4 * 4);
            float4 cd = make_float4(0.f, 0.f, 0.f, 0.f);
            if (kKV && kNorm) cd = *(const float4*)(cold + colbase + e4 * 4);
            const float lcv[4] = {lc.x, lc.y, lc.z, lc.w};
            const float cdv[4] = {cd.x, cd.y, cd.z, cd.w};
            float Pv[4], dSv[4];
#pragma unroll
            for (int z = 0; z < 4; ++z) {
              const int e = e4 * 4 + z, col = colbase + e;
              const float sv = __uint_as_float(rs[e]);
              float dp = __uint_as_float(rd[e]);
              if (kNorm) dp += kKV ? cdv[z] : dden_own;
              const bool valid = kKV ? (col >= own) : (col <= own);
              const float d = kKV ? lcv[z] - l_own : l_own - lcv[z];
              float E = valid ? sig2 * exp2_approx(fminf(d, 0.f)) : 0.f;
              if (kNorm) E *= kKV ? cinv[col & 127] : rinv_own;
              const float T = E * sv;
              Pv[z] = T * sv;
              dSv[z] = dp * T;
              red.x = fmaf(dp, Pv[z], red.x);
            }
            pp[e4 * 2] = pack_bf16(Pv[0], Pv[1]);
            pp[e4 * 2 + 1] = pack_bf16(Pv[2], Pv[3]);
            pd[e4 * 2] = pack_bf16(dSv[0], dSv[1]);
            pd[e4 * 2 + 1] = pack_bf16(dSv[2], dSv[3]);
          }
        }
        // in place: bf16 pairs of columns [cofs, cofs+16) land in u32 columns
        // [32 grp + 8 hh, +8) -- inside this warp's own, already-read range
        if (kKV) tmem_st8(tS + lane_off + grp * 32 + hh * 8, pp);
        tmem_st8(tDP + lane_off + grp * 32 + hh * 8, pd);
      }
      tc_wait_st();
      PA_TR(n * 8 + 6);
      tc_fence_before();
      __syncwarp();
      if (l == 0) mbar_arrive(p_full);
    }
    // epilogue: this warp's 32 gradient columns in fp32 stream-major rows
    mbar_wait(fin, 0);
    tc_fence_after();
    const size_t tokr = (size_t)s * g.t + c0 + own;
    uint32_t r[32];
    tmem_ld32(tA + lane_off + grp * 32, r);
    tc_wait_ld();
    // rows go out through shared memory (the drained operand tiles; 32 rows x 36
    // floats per warp, padded against bank conflicts): each warp store then writes
    // four contiguous 128-byte half-rows instead of 32 scattered 16-byte pieces
    float* stg = (float*)smem + w * (32 * 36);
    const size_t tok0r = (size_t)s * g.t + c0 + own - l;   // row of lane 0
    auto put = [&](float* base, float f) {
#pragma unroll
      for (int a = 0; a < 32; a += 4)
        *(float4*)(stg + l * 36 + a) = make_float4(f * __uint_as_float(r[a]), f * __uint_as_float(r[a + 1]),
                                                   f * __uint_as_float(r[a + 2]), f * __uint_as_float(r[a + 3]));
      __syncwarp();
#pragma unroll
      for (int r4 = 0; r4 < 32; r4 += 4) {
        const int rw = r4 + (l >> 3), cc = (l & 7) * 4;
        *(float4*)(base + (tok0r + rw) * HD + grp * 32 + cc) = *(const float4*)(stg + rw * 36 + cc);
      }
      __syncwarp();
    };
    put(kKV ? out_b : out_a, kKV ? 1.f : 2.f);   // kKV: dV; q-side: dQ (dS carries a factor 1/2)
    if (kKV) {
      tmem_ld32(tB + lane_off + grp * 32, r);
      tc_wait_ld();
      put(out_a, 2.f);   // dK
    }
    // the two column-half warps of a row combine in shared memory (the drained
    // operand tiles) so each token gets one addition per kernel: a fixed order
    float* rsum_s = (float*)smem + 8 * (32 * 36);
    const float rr = red.x + red.y;
    if (grp == 1) rsum_s[row] = rr;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (grp == 0 && g.gated && dell) atomicAdd(dell + tokr, kKV ? -(rr + rsum_s[row]) : rr + rsum_s[row]);
  }
  tc_fence_before();
  __syncthreads();
  if (w == W_TMEM) tmem_dealloc<256>(tm);
}

int tc_intra_bwd_q(const Geo& g, const CUtensorMap& m_q, const CUtensorMap& m_k, const CUtensorMap& m_v,
                   const CUtensorMap& m_dn, const float* ell, const float* dden, const float* rsum, float* dq32,
                   float* dell, cudaStream_t st) {
  using namespace ib2;
  const dim3 grid(g.c / 128, g.n, g.ns);
  auto qs = g.normalize ? k_tc_ib<false, true> : k_tc_ib<false, false>;
  cudaFuncSetAttribute(qs, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  qs<<<grid, THREADS, SMEM, st>>>(m_q, m_k, m_v, m_dn, g, ell, dden, rsum, dq32, nullptr, dell);
  count_launch();
  return 0;
}

}  // namespace pa
