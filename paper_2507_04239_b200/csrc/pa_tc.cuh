// Host-side interface of the bf16 tcgen05 (sm_100a tensor-core) pipeline.
#pragma once
#include <cuda.h>

#include "pa_common.cuh"

namespace pa {

bool tc_supported(const Geo& g, int dtype);
size_t tc_fwd_workspace_bytes(const Geo& g);
size_t tc_bwd_workspace_bytes(const Geo& g);
// mode 0: whole pass.  Sequence-parallel (Geo k0/ng/prefix): mode 1 = local
// phase (forward: end state of this partition from a zero carry -> end_out;
// backward: prefix cotangent from a zero end-state cotangent -> pre_out),
// mode 2 = finish with the incoming carry (state / end-state cotangent).
// Carries are fp32 [ns][2304][80] in the feature-slot order of the states.
int tc_forward(const Geo& g, const void* q, const void* k, const void* v, const float* log_g, void* y,
               float* rowsum, void* ws, cudaStream_t st, int mode = 0, const float* carry = nullptr,
               float* end_out = nullptr);
int tc_backward(const Geo& g, const void* q, const void* k, const void* v, const float* log_g,
                const void* y, const float* rowsum, const void* dy, void* dq, void* dk, void* dv,
                float* dlog_g, const void* fwd_ws, void* bwd_ws, cudaStream_t st, int mode = 0,
                const float* carry = nullptr, float* pre_out = nullptr);
// out = exp(sum of this partition's log lambda) * carry + local (per stream)
int tc_sp_combine(const Geo& g, const void* fwd_ws, const float* carry, const float* local, float* out,
                  cudaStream_t st);
constexpr size_t kSpStateFloatsPerStream = 2304 * 80;

// forward output: intra-chunk attention + state query + combine + normalize (pa_tc_out.cu)
int tc_out(const Geo& g, const CUtensorMap& m_q, const CUtensorMap& m_k, const CUtensorMap& m_v, const void* q,
           const float* ell, const __half* st_main, const __half* st_den, int with_den, void* y, float* rowsum,
           float* y32, int* zflag, cudaStream_t st);

// TMA maps: [b][t][h][64] bf16 with a box of `box_tokens` tokens of one stream;
// row-major [rows][cols] bf16 (fp32 = 0) or fp32 (fp32 = 1) with a bc x br box, SW128
bool tc_map_bth(CUtensorMap* m, const void* ptr, const Geo& g, int box_tokens);
bool tc_map_2d(CUtensorMap* m, const void* ptr, size_t rows, int cols, int bc, int br, int fp32);

// intra-chunk backward in one pass (pa_tc_intra_bwd.cu): dK, dV as bf16 rows
// [ns*t][64], dQ reduce-added into a zeroed fp32 [ns*t][64] (deterministic
// mode: the query side runs as tc_intra_bwd_q instead).  Normalization is
// applied in fp32 from dden and the forward rowsum.  Log-gate cotangents:
// dell += (zeroed by the caller).
int tc_intra_bwd_fused(const Geo& g, const void* q, const void* k, const void* v, const void* dy, const float* ell,
                       const float* dden, const float* rsum, __nv_bfloat16* dk16, __nv_bfloat16* dv16, float* dq32,
                       float* dell, cudaStream_t st);
// query side alone (pa_tc_ib.cu; fixed accumulation order): dq32 (=), the
// query-side log-gate cotangents (dell +=, one addition per token)
int tc_intra_bwd_q(const Geo& g, const CUtensorMap& m_q, const CUtensorMap& m_k, const CUtensorMap& m_v,
                   const CUtensorMap& m_dn, const float* ell, const float* dden, const float* rsum, float* dq32,
                   float* dell, cudaStream_t st);

// expanded-state VJP GEMMs (pa_tc_zvjp.cu): E = expanded A'_{k-1} (query side) or dS~_k (update side)
int tc_zvjp(const Geo& g, bool upd, int u_bf16_bth, const void* u_rows, const __half* u16, const void* xraw,
            const float* ell, const float* lamlog, const __half* E, const void* dx32, const void* dv32,
            float* dell, float* dellend, void* dxo, void* dvo, cudaStream_t st);

}  // namespace pa
