/*
 * power_attention_b200.h -- C ABI of the B200-native chunked power attention.
 *
 * Plain pointers, sizes and a cudaStream_t; no torch types.  Every pointer is
 * device memory unless stated otherwise.  All entry points are stream-ordered
 * and asynchronous (no host synchronisation), reentrant, and return 0 on
 * success or a PA_ERR_* code (message via pa_last_error(), thread-local).
 *
 * Tensor layout is the reference's [b, t, h, x] (row-major, contiguous):
 *   q, k : [b, t, h, d]     v, y : [b, t, h, e]     log_g, rowsum : [b, t, h]
 * ("e" is the value width, the reference's "v").
 *
 * Reference interfaces replaced (file:line under /root/reference/pkg/src/power_attention):
 *   pa_update_state   <- _core.update_state   _core.pyx:18-43  (dispatch kernels.py:55-83)
 *   pa_query_state    <- _core.query_state    _core.pyx:46-64  (dispatch kernels.py:86-110)
 *   pa_discumsum      <- discumsum            chunked.py:156-176
 *   pa_power_full_fwd <- chunked_power_attention chunked.py:287-413 (attention form when chunk >= t,
 *                        attention.py:273-309), with log-gates g = exp(log_g)
 *   pa_power_full_bwd <- vjp_chunked          gradients.py:361-483 (dlog_g = g * dgates)
 *   pa_power_logspace_fwd <- power_attention_form use_log_space branch attention.py:289-305
 *   pa_feature_dim / pa_feature_table <- expansion_dim / monomial_table expansions.py:87-99, 171-198
 */
#ifndef POWER_ATTENTION_B200_H
#define POWER_ATTENTION_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* pa_stream_t; /* == cudaStream_t */

enum pa_dtype { PA_F32 = 0, PA_BF16 = 1, PA_F16 = 2, PA_F64 = 3 };

enum pa_status {
  PA_OK = 0,
  PA_ERR_INVALID_SPEC = 1,   /* -> errors.InvalidSpec          (errors.py:8)  */
  PA_ERR_SHAPE = 2,          /* -> errors.ShapeMismatch        (errors.py:16) */
  PA_ERR_CUDA = 3,           /* CUDA launch / runtime failure                  */
  PA_ERR_UNSUPPORTED = 4,    /* shape/dtype outside what the kernels cover    */
  PA_ERR_WORKSPACE = 5,      /* workspace smaller than pa_*_workspace_bytes   */
  PA_ERR_ODD_NORMALIZE = 6   /* -> errors.OddPowerWithNormalize (errors.py:24) */
};

/* Behaviour flags (pa_problem.flags). */
enum pa_flags {
  /* Fixed accumulation order: every tensor-core accumulator is fed by one MMA
   * issuer in a fixed order, so repeated calls are bit-identical (slower). */
  PA_FLAG_DETERMINISTIC = 1,
  /* Refuse (PA_ERR_UNSUPPORTED) instead of running a 16-bit problem on the fp32
   * CUDA-core kernels when the tensor-core kernels do not cover its shape. */
  PA_FLAG_STRICT_TC = 2,
  /* Sequence-parallel / streaming states always carry the key-sum column (the
   * reference ChunkState.key_sum), also when the call does not normalize. */
  PA_FLAG_KEY_SUM = 4
};

/* One power_full problem (reference AttentionConfig attention.py:106-171 +
 * ChunkPlan chunked.py:66-86). */
typedef struct pa_problem {
  int32_t b, t, h, d, e; /* batch, tokens, heads, q/k width, value width      */
  int32_t p;             /* degree of the SPOW_p expansion (1..4)             */
  int32_t chunk;         /* chunk size c; c >= t selects the attention form   */
  int32_t normalize;     /* 1: divide by the score sum (even p only)          */
  int32_t dtype;         /* pa_dtype of q, k, v, y, dy, dq, dk, dv            */
  int32_t gated;         /* 1: log_g is read; 0: ungated (log_g ignored)      */
  int32_t has_scale;     /* 1: use `scale` exactly (any sign); 0: 1/sqrt(d)   */
  int32_t flags;         /* pa_flags                                          */
  double scale;          /* sigma (attention.py:149-150), when has_scale      */
} pa_problem;

/* 1 when the problem runs on the tcgen05 tensor-core kernels (p = 2), 2 when
 * its state GEMMs do (the degree-4 path: bf16, p = 4, d = e = 32), 0 when it
 * runs on the fp32 CUDA-core kernels, negative PA_ERR_* when it is invalid. */
int pa_uses_tensor_cores(const pa_problem* pr);

/* Expansion kinds (reference expansions.py:41-44). */
enum pa_expansion { PA_SPOW = 0, PA_TPOW = 1, PA_TSPOW = 2 };
/* D of an expansion (d_tile only for TSPOW, must divide d); -1 if invalid.
 * Reference expansion_dim expansions.py:87-99. */
int64_t pa_expansion_dim(int32_t kind, int32_t p, int32_t d, int32_t d_tile);
/* Host buffers idx [D*p] int32, w [D] double: the reference monomial_table
 * (expansions.py:171-198) for SPOW, TPOW or TSPOW, same row order. */
int pa_expansion_table(int32_t kind, int32_t p, int32_t d, int32_t d_tile, int32_t* idx, double* w);

/* D = C(d+p-1, p); -1 on overflow. */
int64_t pa_feature_dim(int32_t p, int32_t d);
/* Host buffers: idx [D*p] int32 (NDMI, lexicographic), w [D] double. */
int pa_feature_table(int32_t p, int32_t d, int32_t* idx, double* w);

/* Bytes of forward workspace.  The forward leaves in it everything the
 * backward needs; keep it alive between the two calls. */
size_t pa_fwd_workspace_bytes(const pa_problem* pr);
size_t pa_bwd_workspace_bytes(const pa_problem* pr);

/* y [b,t,h,e] (dtype), rowsum [b,t,h] fp32 (may be NULL). */
int pa_power_full_fwd(const pa_problem* pr, const void* q, const void* k, const void* v,
                      const float* log_g, void* y, float* rowsum, void* ws, size_t ws_bytes,
                      pa_stream_t stream);

/* Gradients for a cotangent dy on y.  y and rowsum are the forward outputs
 * (rowsum required when normalize=1).  dlog_g [b,t,h] fp32 (NULL if ungated). */
int pa_power_full_bwd(const pa_problem* pr, const void* q, const void* k, const void* v,
                      const float* log_g, const void* y, const float* rowsum, const void* dy,
                      void* dq, void* dk, void* dv, float* dlog_g, const void* fwd_ws,
                      void* bwd_ws, size_t bwd_ws_bytes, pa_stream_t stream);

/* Log-space (stabilised) attention form, reference attention.py:289-305
 * (power_attention_form with use_log_space; even p only): scores
 * p*log(|s|+eps) + log-decay, row-max shifted, exponentiated.  q, k, v, y of
 * `pr->dtype` (F32 or F64), log_g and rowsum [b,t,h] of the same dtype (log_g
 * may hold -inf for zero gates; NULL when ungated).  pr->chunk is ignored (one
 * chunk spans the sequence); t <= 16384, e <= 128.  No workspace. */
int pa_power_logspace_fwd(const pa_problem* pr, double eps, const void* q, const void* k,
                          const void* v, const void* log_g, void* y, void* rowsum,
                          pa_stream_t stream);

/* ---------------------------------------------------------------- sequence parallel
 * A sequence split into contiguous chunk ranges, one per rank (
 * the reference runs the discumsum of chunked.py:356-367 serially over all
 * chunks).  discumsum is a linear recurrence with the associative combine
 * (l1, S1) o (l2, S2) = (l1 l2, l2 S1 + S2), so each rank runs:
 *   fwd: pa_sp_fwd_local -> E_r (its end state from a zero carry);
 *        carry chain: C_0 = 0, C_{r+1} = pa_sp_combine(C_r, E_r)  (rank-to-rank P2P);
 *        pa_sp_fwd_finish(C_r) -> y
 *   bwd: pa_sp_bwd_local -> P_r (cotangent of its incoming state from a zero carry);
 *        reverse chain: H_{R-1} = 0, H_{r-1} = pa_sp_combine(H_r, P_r);
 *        pa_sp_bwd_finish(H_r) -> dq, dk, dv, dlog_g
 * Carries are fp32 [b*h][2304][80] (pa_sp_state_floats), zero-initialised by
 * the caller.  Tensor-core path only (bf16, p = 2, d = e = 64, t % chunk == 0). */
typedef struct pa_sp_part {
  int32_t chunk0;  /* global index of this rank's first chunk                    */
  int32_t nchunks; /* chunks of the whole sequence                              */
} pa_sp_part;

size_t pa_sp_state_floats(const pa_problem* pr);
int pa_sp_fwd_local(const pa_problem* pr, const pa_sp_part* sp, const void* q, const void* k, const void* v,
                    const float* log_g, void* ws, size_t ws_bytes, float* end_state, pa_stream_t stream);
int pa_sp_fwd_finish(const pa_problem* pr, const pa_sp_part* sp, const void* q, const void* k, const void* v,
                     const float* log_g, void* y, float* rowsum, void* ws, size_t ws_bytes, const float* carry,
                     pa_stream_t stream);
int pa_sp_bwd_local(const pa_problem* pr, const pa_sp_part* sp, const void* q, const void* k, const void* v,
                    const float* log_g, const void* y, const float* rowsum, const void* dy, const void* fwd_ws,
                    void* bwd_ws, size_t bwd_ws_bytes, float* prefix_cot, pa_stream_t stream);
int pa_sp_bwd_finish(const pa_problem* pr, const pa_sp_part* sp, const void* q, const void* k, const void* v,
                     const float* log_g, const void* y, const float* rowsum, const void* dy, void* dq, void* dk,
                     void* dv, float* dlog_g, const void* fwd_ws, void* bwd_ws, size_t bwd_ws_bytes,
                     const float* carry_cot, pa_stream_t stream);
/* out = exp(sum of this rank's chunk log-decays) * carry + local, per stream
 * (carry may be NULL = zero).  Needs the rank's forward workspace. */
int pa_sp_combine(const pa_problem* pr, const pa_sp_part* sp, const void* fwd_ws, const float* carry,
                  const float* local, float* out, pa_stream_t stream);

/* Device-side status of the last forward: number of non-positive score sums
 * seen while normalizing (the reference raises ZeroDenominator,
 * chunked.py:392-395).  Reads 4 bytes from ws; synchronises the stream. */
int pa_fwd_zero_denominators(const pa_problem* pr, const void* ws, pa_stream_t stream,
                             int32_t* count);

/* Reference _core.update_state: state[s] (+)= sum_j w[s,j] phi(k[s,j]) (x) v[s,j],
 * key_sum[s] (+)= sum_j w[s,j] phi(k[s,j]).  k [n,c,d], v [n,c,e], w [n,c] or
 * NULL (all ones), state [n,D,e], key_sum [n,D]; all of `dtype` (F32 or F64).
 * accumulate=0 overwrites, 1 adds (the reference accumulates into zeroed
 * outputs). */
int pa_update_state(int32_t n, int32_t c, int32_t d, int32_t e, int32_t p, int32_t dtype,
                    const void* k, const void* v, const void* w, void* state, void* key_sum,
                    int32_t accumulate, pa_stream_t stream);

/* Reference _core.query_state: y[s,m] (+)= phi(q[s,m]) . state[s],
 * denom[s,m] (+)= phi(q[s,m]) . key_sum[s]; q pre-scaled [n,c,d]. */
int pa_query_state(int32_t n, int32_t c, int32_t d, int32_t e, int32_t p, int32_t dtype,
                   const void* q, const void* state, const void* key_sum, void* y, void* denom,
                   int32_t accumulate, pa_stream_t stream);

/* The same two operators with the caller's monomial table (the reference
 * _core ABI passes idx and weights too, _core.pyx:18-20, 46-48), so any
 * expansion kind runs: idx [D*p] int32 and weights [D] f64 in DEVICE memory
 * (pa_expansion_table fills host buffers).  p <= 4. */
int pa_update_state_table(int32_t n, int32_t c, int32_t d, int32_t e, int32_t p, int64_t D, int32_t dtype,
                          const void* k, const void* v, const void* w, const int32_t* idx, const double* weights,
                          void* state, void* key_sum, int32_t accumulate, pa_stream_t stream);
int pa_query_state_table(int32_t n, int32_t c, int32_t d, int32_t e, int32_t p, int64_t D, int32_t dtype,
                         const void* q, const void* state, const void* key_sum, const int32_t* idx,
                         const double* weights, void* y, void* denom, int32_t accumulate, pa_stream_t stream);

/* Reference discumsum: out[0] = values[0]; out[k] = lams[k-1, l] * out[k-1, l, m]
 * + values[k, l, m] with a separate multiply and add (bit-exact with the
 * sequential loop).  values/out [n, L, M]; lams [n-1, L]; out may alias values. */
int pa_discumsum(int32_t n, int64_t L, int64_t M, int32_t dtype, const void* values,
                 const void* lams, void* out, pa_stream_t stream);

/* Per-stage device timing: CUDA events recorded on the launching stream
 * around every kernel of the pipelines while enabled.  pa_profile_read fills
 * up to cap entries (names: cap x 32 bytes) with accumulated milliseconds and
 * launch counts per stage and returns the number of entries (synchronises). */
int pa_profile_enable(int32_t on);
void pa_profile_reset(void);
int pa_profile_read(char* names, double* ms, int64_t* launches, int32_t cap);

const char* pa_last_error(void);
/* Number of CUDA kernels this library launched since load (for the bench's
 * gpu_launches claim). */
int64_t pa_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
