// Host-side interface of the fp32 CUDA-core kernels (pa_simt.cu).
#pragma once
#include "pa_common.cuh"

namespace pa {

struct SimtWs {           // forward workspace, kept for the backward
  float* ell;             // [ns, t]
  float* lamlog;          // [ns, n]
  int* idx;               // [D, p]
  float* wt;              // [D]
  float* A;               // [ns, n, D, E1]
  float* yat;             // [ns, t, E1]
  int* zflag;             // [1]
  float* y32;             // [ns, t, e] normalized output in fp32 (normalize only)
  char* tc4;              // scratch of the degree-4 tensor-core state GEMMs (pa_tc4.cu), or empty
};

// degree-4 state GEMMs on the tensor cores (pa_tc4.cu): bf16, p = 4, d = e = 32
bool tc4_supported(const Geo& g, int dtype);
size_t tc4_extra_bytes(const Geo& g);
// out [ns, n, D, e+1] (fwd: S_k from x = k, v; bwd: dA of slot k-1 from x = q, dz)
int tc4_state(const Geo& g, bool bwd, const void* x, const void* v, const float* dz, const float* ell,
              const float* lamlog, const int* idx, const float* wt, void* scratch, float* out, cudaStream_t st);
// slot count of the degree-4 block order; copies its (idx, wt) table into a workspace
int tc4_slots();
int tc4_copy_tables(int* idx, float* wt, cudaStream_t st);
unsigned* tc4_mxs(const Geo& g, void* scratch);  // per-chunk maxima recorded by tc4_state
// degree-4 intra-chunk attention on the tensor cores; 1 = shape not covered
int tc4_intra_fwd(const Geo& g, const void* q, const void* k, const void* v, const float* ell, float* yat,
                  void* scratch, cudaStream_t st);
// its VJP (needs the padded copies of tc4_intra_fwd in the same scratch); 1 = not covered
int tc4_intra_bwd(const Geo& g, const float* ell, const float* dz, const void* dy, const float* rowsum, float* dq32,
                  float* dk32, float* dv32, float* dell, void* scratch, cudaStream_t st);
// discumsum fused with the fp16 operand conversion (pa_tc4.cu)
int tc4_scan_fwd(const Geo& g, const float* lamlog, float* A, const float* wt, void* scratch, cudaStream_t st);
int tc4_scan_bwd(const Geo& g, const float* lamlog, const float* A, const float* dA, float* dlam, const float* wt,
                 void* scratch, cudaStream_t st);
int tc4_vjp(const Geo& g, bool upd, const void* x, float* dx32, float* dell, float* dellend, void* scratch,
            cudaStream_t st);
int tc4_tok(const Geo& g, int mode, const void* x, const float* ell, const float* lamlog, const float* yat, void* y,
            float* rowsum, float* y32, int* zflag, float* dv32, void* scratch, cudaStream_t st);

struct SimtBwdWs {
  float* dz;              // [ns, t, E1]
  float* dA;              // [ns, n, D, E1]
  float* dq32;            // [ns, t, d]
  float* dk32;            // [ns, t, d]
  float* dv32;            // [ns, t, e]
  float* dell;            // [ns, t]
  float* dellend;         // [ns, n]
  float* dlam;            // [ns, n]
};

int64_t host_binom(int64_t n, int64_t k);
size_t simt_fwd_bytes(const Geo& g);
size_t simt_bwd_bytes(const Geo& g);
SimtWs simt_carve_fwd(const Geo& g, void* ws);
SimtBwdWs simt_carve_bwd(const Geo& g, void* ws);
void host_feature_table(int p, int d, int* idx, double* w);
// kind 0 = SPOW, 1 = TPOW, 2 = TSPOW (tile edge d_tile)
int64_t host_expansion_dim(int kind, int p, int d, int d_tile);
void host_expansion_table(int kind, int p, int d, int d_tile, int* idx, double* w);
int simt_build_table(int p, int d, int D, int* idx, float* wt, cudaStream_t st);
int simt_forward(const Geo& g, int dtype, const void* q, const void* k, const void* v, const float* lg,
                 void* y, float* rs, const SimtWs& w, cudaStream_t st);
int simt_backward(const Geo& g, int dtype, const void* q, const void* k, const void* v, const void* y,
                  const float* rs, const void* dy, void* dq, void* dk, void* dv, float* dlogg,
                  const SimtWs& w, const SimtBwdWs& b, cudaStream_t st);
int simt_intra_bwd(const Geo& g, const __nv_bfloat16* q, const __nv_bfloat16* k, const __nv_bfloat16* v,
                   const float* ell, const float* dz, float* dq32, float* dk32, float* dv32, float* dell,
                   cudaStream_t st);
int simt_gate_finish(const Geo& g, const float* lamlog, const float* dell, const float* dellend,
                     const float* dlam, float* dlogg, cudaStream_t st);
int simt_finalize_bf16(const Geo& g, const float* src, int w, void* dst, cudaStream_t st);
int pub_update(int n, int c, int d, int e, int p, int D, int dtype, const void* k, const void* v,
               const void* w, const int* idx, const double* wt, void* state, void* ks, int acc,
               cudaStream_t st);
int pub_query(int n, int c, int d, int e, int p, int D, int dtype, const void* q, const void* state,
              const void* ks, const int* idx, const double* wt, void* y, void* den, int acc, cudaStream_t st);
int pub_discumsum(int n, int64_t L, int64_t M, int dtype, const void* values, const void* lams, void* out,
                  cudaStream_t st);

}  // namespace pa
