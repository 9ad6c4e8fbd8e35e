// C ABI (include/power_attention_b200.h): validation, workspace carving and
// the stage order of the forward / backward pipelines.
#include <math.h>

#include <string.h>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/power_attention_b200.h"
#include "pa_common.cuh"
#include "pa_simt.cuh"
#include "pa_tc.cuh"

namespace pa {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return PA_ERR_CUDA;
  }
  return PA_OK;
}

// ---------------------------------------------------------------- profiling
struct ProfRec {
  const char* name;
  cudaEvent_t a, b;
};
static std::mutex g_pm;
static std::vector<ProfRec> g_prof;
static std::atomic<bool> g_prof_on{false};
static std::map<std::string, std::pair<double, int64_t>> g_prof_acc;

StageTimer::StageTimer(const char* n, cudaStream_t s) : name(n), st(s), a(nullptr) {
  if (!g_prof_on.load()) return;
  cudaEventCreate(&a);
  cudaEventRecord(a, st);
}
StageTimer::~StageTimer() {
  if (!a) return;
  cudaEvent_t b;
  cudaEventCreate(&b);
  cudaEventRecord(b, st);
  std::lock_guard<std::mutex> lk(g_pm);
  g_prof.push_back({name, a, b});
}

static void prof_drain() {
  std::lock_guard<std::mutex> lk(g_pm);
  for (auto& r : g_prof) {
    float ms = 0.f;
    cudaEventSynchronize(r.b);
    cudaEventElapsedTime(&ms, r.a, r.b);
    auto& e = g_prof_acc[r.name];
    e.first += ms;
    e.second += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
}

static size_t align_up(size_t x) { return (x + 255) & ~size_t(255); }

// Carves consecutive 256-byte aligned regions out of one workspace buffer.
struct Carver {
  char* base;
  size_t off = 0;
  explicit Carver(void* b) : base((char*)b) {}
  template <typename T>
  T* take(size_t count) {
    T* p = base ? (T*)(base + off) : nullptr;
    off += align_up(count * sizeof(T));
    return p;
  }
};

static int make_geo(const pa_problem* pr, Geo* g) {
  if (!pr) {
    set_error("null problem");
    return PA_ERR_INVALID_SPEC;
  }
  if (pr->b < 1 || pr->t < 1 || pr->h < 1 || pr->d < 1 || pr->e < 1) {
    set_error("need b, t, h, d, e >= 1");
    return PA_ERR_SHAPE;
  }
  if (pr->p < 1 || pr->p > 4) {
    set_error("power degree p must be in [1, 4] on the CUDA path");
    return PA_ERR_UNSUPPORTED;
  }
  if (pr->d > 128 || pr->e > 128) {
    set_error("d and e must be <= 128 on the CUDA path");
    return PA_ERR_UNSUPPORTED;
  }
  if (pr->chunk < 1) {
    set_error("chunk_size must be >= 1");
    return PA_ERR_INVALID_SPEC;
  }
  if (pr->normalize && (pr->p % 2)) {
    set_error("normalization needs positive scores: p must be even");
    return PA_ERR_ODD_NORMALIZE;
  }
  if (pr->dtype < 0 || pr->dtype > 2) {
    set_error("power_full dtype must be f32, bf16 or f16");
    return PA_ERR_UNSUPPORTED;
  }
  g->b = pr->b;
  g->t = pr->t;
  g->h = pr->h;
  g->d = pr->d;
  g->e = pr->e;
  g->E1 = pr->e + 1;
  g->p = pr->p;
  g->c = std::min(pr->chunk, pr->t);
  g->n = (pr->t + g->c - 1) / g->c;
  int64_t D = host_binom(pr->d + pr->p - 1, pr->p);
  if (D > (int64_t)1 << 30) {
    set_error("expanded dimension too large");
    return PA_ERR_UNSUPPORTED;
  }
  g->D = (int)D;
  g->ns = pr->b * pr->h;
  g->scale = pr->has_scale ? (float)pr->scale : 1.0f / sqrtf((float)pr->d);
  g->det = (pr->flags & PA_FLAG_DETERMINISTIC) ? 1 : 0;
  g->keysum = (pr->flags & PA_FLAG_KEY_SUM) ? 1 : 0;
  g->normalize = pr->normalize ? 1 : 0;
  g->gated = pr->gated ? 1 : 0;
  g->bth = 1;
  g->k0 = 0;
  g->ng = g->n;
  g->prefix = 0;
  g->nsl = g->n + 1;
  g->treal = g->t;
  g->dtype = pr->dtype;
  // the degree-4 tensor-core path orders features in blocks of four (pa_tc4.cu):
  // its states hold tc4_slots() rows (zero-weight duplicates included)
  if (tc4_supported(*g, pr->dtype)) g->D = tc4_slots();
  return PA_OK;
}

// The tensor-core path serves every bf16 / fp16 problem with p = 2, d = e = 64.
// Its kernels want a chunk that is a multiple of 128 up to 1024 and t a multiple
// of the chunk; the caller's shape maps onto that as follows.
//  * Chunk size: the outputs and gradients of chunked power attention do not
//    depend on the chunk size (the reference's own test, test_chunked.py:278-285,
//    holds them equal to 2e-8 in f64); a chunk the kernels do not take runs with
//    an internal chunk of min(1024, t rounded up to 128) -- only rounding differs.
//  * A partial last chunk (reference ChunkPlan.bounds chunked.py:85-86 ends it
//    early) runs on a zero-padded copy: padded keys and values are zero and padded
//    log-gates 0, so the padding adds nothing to any real token's output, state or
//    gradient; padded rows are dropped (normalized: weight 0, Geo.treal).
//  * fp16 inputs are staged as bf16 (one rounding, 2^-9) and the outputs and
//    gradients converted back.
// Returns false when the tensor-core path does not apply.  `stage` = the call
// runs on copies in the workspace (padding or fp16).
static bool tc_geo(const pa_problem* pr, const Geo& g, Geo* gp, bool* stage) {
  if (pr->dtype != PA_BF16 && pr->dtype != PA_F16) return false;
  Geo p = g;
  const bool chunk_ok = g.c % 128 == 0 && g.c <= 1024;
  if (!chunk_ok) p.c = std::min(1024, (g.t + 127) / 128 * 128);
  p.t = (g.t + p.c - 1) / p.c * p.c;
  p.n = p.t / p.c;
  p.nsl = p.n + 1;
  p.ng = p.n;
  p.treal = g.t;
  p.dtype = PA_BF16;
  if (!tc_supported(p, PA_BF16)) return false;
  *gp = p;
  *stage = p.t != g.t || pr->dtype == PA_F16;
  return true;
}

// Which kernel family runs the problem (g becomes the tensor-core geometry when
// that path applies); with PA_FLAG_STRICT_TC a 16-bit problem the tensor-core
// kernels do not cover is an error, not a silent switch to the fp32 CUDA-core
// kernels.
static int route(const pa_problem* pr, Geo& g, bool* tc, bool* stage = nullptr) {
  Geo gp;
  bool st = false;
  *tc = tc_geo(pr, g, &gp, &st);
  if (*tc) g = gp;
  if (stage) *stage = st;
  if (!*tc && !tc4_supported(g, pr->dtype) && (pr->flags & PA_FLAG_STRICT_TC) && pr->dtype != PA_F32) {
    set_error("strict tensor-core mode: the tcgen05 kernels cover bf16 / fp16 with p = 2, d = e = 64, and bf16 "
              "with p = 4, d = e = 32");
    return PA_ERR_UNSUPPORTED;
  }
  return PA_OK;
}

constexpr int HDIM = 64;

// fp16 <-> bf16 staging with the zero tail: dst rows [b][t_dst][h][64], src rows
// [b][t_src][h][64]; rows past t_src are zero
template <typename TD, typename TS>
__global__ void k_stage_rows(TD* dst, const TS* src, int b, int t_dst, int t_src, int hw) {
  const size_t per = (size_t)t_dst * hw, tot = (size_t)b * per;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < tot; i += (size_t)gridDim.x * blockDim.x) {
    const size_t bi = i / per, r = i - bi * per;
    float v = 0.f;
    if (r < (size_t)t_src * hw) v = to_f<TS>(src[bi * (size_t)t_src * hw + r]);
    dst[i] = from_f<TD>(v);
  }
}
static void stage_rows(void* dst, const void* src, const Geo& g, int to_bf16, size_t t_dst, size_t t_src,
                       cudaStream_t st) {
  const int hw = g.h * HDIM;
  const size_t tot = (size_t)g.b * t_dst * hw;
  const unsigned blocks = (unsigned)std::min<size_t>((tot + 255) / 256, 148 * 16);
  if (to_bf16)
    k_stage_rows<__nv_bfloat16, __half><<<blocks, 256, 0, st>>>((__nv_bfloat16*)dst, (const __half*)src, g.b,
                                                                 (int)t_dst, (int)t_src, hw);
  else
    k_stage_rows<__half, __nv_bfloat16><<<blocks, 256, 0, st>>>((__half*)dst, (const __nv_bfloat16*)src, g.b,
                                                                 (int)t_dst, (int)t_src, hw);
  count_launch();
}

// zero-padded copies for the padded tensor-core path: per batch, t real rows of
// `rb` bytes then t_pad - t zero rows
struct PadFwd {
  char *q, *k, *v, *y;
  float *lg, *rs;
};
struct PadBwd {
  char *dy, *dq, *dk, *dv;
  float* dlg;
};
static PadFwd carve_pad_fwd(const Geo& g, void* base, size_t* bytes) {
  Carver c(base);
  PadFwd p;
  const size_t rows = (size_t)g.b * g.t * g.h;
  p.q = c.take<char>(rows * g.d * 2);
  p.k = c.take<char>(rows * g.d * 2);
  p.v = c.take<char>(rows * g.e * 2);
  p.y = c.take<char>(rows * g.e * 2);
  p.lg = c.take<float>(rows);
  p.rs = c.take<float>(rows);
  *bytes = c.off;
  return p;
}
static PadBwd carve_pad_bwd(const Geo& g, void* base, size_t* bytes) {
  Carver c(base);
  PadBwd p;
  const size_t rows = (size_t)g.b * g.t * g.h;
  p.dy = c.take<char>(rows * g.e * 2);
  p.dq = c.take<char>(rows * g.d * 2);
  p.dk = c.take<char>(rows * g.d * 2);
  p.dv = c.take<char>(rows * g.e * 2);
  p.dlg = c.take<float>(rows);
  *bytes = c.off;
  return p;
}
static void pad_rows(void* dst, const void* src, const Geo& g, size_t row_bytes, cudaStream_t st) {
  const size_t rb = (size_t)g.h * row_bytes;   // one token of every head
  cudaMemcpy2DAsync(dst, g.t * rb, src, g.treal * rb, g.treal * rb, g.b, cudaMemcpyDeviceToDevice, st);
  cudaMemset2DAsync((char*)dst + g.treal * rb, g.t * rb, 0, (g.t - g.treal) * rb, g.b, st);
}
static void unpad_rows(void* dst, const void* src, const Geo& g, size_t row_bytes, cudaStream_t st) {
  const size_t rb = (size_t)g.h * row_bytes;
  cudaMemcpy2DAsync(dst, g.treal * rb, src, g.t * rb, g.treal * rb, g.b, cudaMemcpyDeviceToDevice, st);
}
// copy rows into / out of the staged (padded, bf16) layout
static void stage_in(void* dst, const void* src, const Geo& g, int dtype, cudaStream_t st) {
  if (dtype == PA_F16) stage_rows(dst, src, g, 1, g.t, g.treal, st);
  else pad_rows(dst, src, g, (size_t)HDIM * 2, st);
}
static void stage_out(void* dst, const void* src, const Geo& g, int dtype, cudaStream_t st) {
  if (dtype == PA_F16) stage_rows(dst, src, g, 0, g.treal, g.t, st);
  else unpad_rows(dst, src, g, (size_t)HDIM * 2, st);
}
static size_t inner_fwd_bytes(const Geo& g) { return align_up(tc_fwd_workspace_bytes(g)); }
static size_t inner_bwd_bytes(const Geo& g) { return align_up(tc_bwd_workspace_bytes(g)); }

SimtWs carve_simt_fwd(const Geo& g, void* ws, size_t* bytes) {
  Carver c(ws);
  SimtWs w;
  w.zflag = c.take<int>(1);
  w.ell = c.take<float>((size_t)g.ns * g.t);
  w.lamlog = c.take<float>((size_t)g.ns * g.n);
  w.idx = c.take<int>((size_t)g.D * g.p);
  w.wt = c.take<float>(g.D);
  w.A = c.take<float>((size_t)g.ns * g.n * g.D * g.E1);
  w.yat = c.take<float>((size_t)g.ns * g.t * g.E1);
  w.y32 = c.take<float>(g.normalize ? (size_t)g.ns * g.t * g.e : 0);
  w.tc4 = c.take<char>(tc4_supported(g, g.dtype) ? tc4_extra_bytes(g) : 0);
  *bytes = c.off;
  return w;
}

SimtBwdWs carve_simt_bwd(const Geo& g, void* ws, size_t* bytes) {
  Carver c(ws);
  SimtBwdWs b;
  b.dz = c.take<float>((size_t)g.ns * g.t * g.E1);
  b.dA = c.take<float>((size_t)g.ns * g.n * g.D * g.E1);
  b.dq32 = c.take<float>((size_t)g.ns * g.t * g.d);
  b.dk32 = c.take<float>((size_t)g.ns * g.t * g.d);
  b.dv32 = c.take<float>((size_t)g.ns * g.t * g.e);
  b.dell = c.take<float>((size_t)g.ns * g.t);
  b.dellend = c.take<float>((size_t)g.ns * g.n);
  b.dlam = c.take<float>((size_t)g.ns * g.n);
  *bytes = c.off;
  return b;
}

size_t simt_fwd_bytes(const Geo& g) {
  size_t n;
  carve_simt_fwd(g, nullptr, &n);
  return n;
}
size_t simt_bwd_bytes(const Geo& g) {
  size_t n;
  carve_simt_bwd(g, nullptr, &n);
  return n;
}
SimtWs simt_carve_fwd(const Geo& g, void* ws) {
  size_t n;
  return carve_simt_fwd(g, ws, &n);
}
SimtBwdWs simt_carve_bwd(const Geo& g, void* ws) {
  size_t n;
  return carve_simt_bwd(g, ws, &n);
}

}  // namespace pa

using namespace pa;

extern "C" {

int64_t pa_feature_dim(int32_t p, int32_t d) {
  if (p < 1 || d < 1) return -1;
  return host_binom((int64_t)d + p - 1, p);
}

int pa_feature_table(int32_t p, int32_t d, int32_t* idx, double* w) {
  if (p < 1 || p > 4 || d < 1 || !idx || !w) {
    set_error("feature table needs 1 <= p <= 4, d >= 1 and output buffers");
    return PA_ERR_INVALID_SPEC;
  }
  host_feature_table(p, d, idx, w);
  return PA_OK;
}

int pa_uses_tensor_cores(const pa_problem* pr) {
  Geo g;
  if (int rc = make_geo(pr, &g)) return -rc;
  bool tc;
  if (int rc = route(pr, g, &tc)) return -rc;
  if (tc) return 1;
  return tc4_supported(g, pr->dtype) ? 2 : 0;
}

size_t pa_fwd_workspace_bytes(const pa_problem* pr) {
  Geo g;
  if (make_geo(pr, &g)) return 0;
  bool tc, stage;
  if (route(pr, g, &tc, &stage)) return 0;
  if (tc && stage) {
    size_t extra;
    carve_pad_fwd(g, nullptr, &extra);
    return inner_fwd_bytes(g) + extra;
  }
  if (tc) return tc_fwd_workspace_bytes(g);
  size_t n;
  carve_simt_fwd(g, nullptr, &n);
  return n;
}

size_t pa_bwd_workspace_bytes(const pa_problem* pr) {
  Geo g;
  if (make_geo(pr, &g)) return 0;
  bool tc, stage;
  if (route(pr, g, &tc, &stage)) return 0;
  if (tc && stage) {
    size_t extra;
    carve_pad_bwd(g, nullptr, &extra);
    return inner_bwd_bytes(g) + extra;
  }
  if (tc) return tc_bwd_workspace_bytes(g);
  size_t n;
  carve_simt_bwd(g, nullptr, &n);
  return n;
}

int pa_power_full_fwd(const pa_problem* pr, const void* q, const void* k, const void* v,
                      const float* log_g, void* y, float* rowsum, void* ws, size_t ws_bytes,
                      pa_stream_t stream) {
  Geo g;
  if (int rc = make_geo(pr, &g)) return rc;
  if (!q || !k || !v || !y || !ws || (g.gated && !log_g)) {
    set_error("null tensor pointer");
    return PA_ERR_INVALID_SPEC;
  }
  cudaStream_t st = (cudaStream_t)stream;
  bool tc, stage;
  if (int rc = route(pr, g, &tc, &stage)) return rc;
  if (tc && stage) {
    size_t extra;
    PadFwd p = carve_pad_fwd(g, (char*)ws + inner_fwd_bytes(g), &extra);
    if (ws_bytes < inner_fwd_bytes(g) + extra) {
      set_error("forward workspace too small");
      return PA_ERR_WORKSPACE;
    }
    stage_in(p.q, q, g, pr->dtype, st);
    stage_in(p.k, k, g, pr->dtype, st);
    stage_in(p.v, v, g, pr->dtype, st);
    if (g.gated) pad_rows(p.lg, log_g, g, 4, st);
    const bool rs = rowsum || g.normalize;
    if (int rc = tc_forward(g, p.q, p.k, p.v, g.gated ? p.lg : nullptr, p.y, rs ? p.rs : nullptr, ws, st)) return rc;
    stage_out(y, p.y, g, pr->dtype, st);
    if (rowsum) unpad_rows(rowsum, p.rs, g, 4, st);
    return cuda_check("padded forward");
  }
  if (tc) {
    if (ws_bytes < tc_fwd_workspace_bytes(g)) {
      set_error("forward workspace too small");
      return PA_ERR_WORKSPACE;
    }
    return tc_forward(g, q, k, v, log_g, y, rowsum, ws, st);
  }
  size_t need;
  SimtWs w = carve_simt_fwd(g, ws, &need);
  if (ws_bytes < need) {
    set_error("forward workspace too small");
    return PA_ERR_WORKSPACE;
  }
  cudaMemsetAsync(w.zflag, 0, sizeof(int), st);
  if (tc4_supported(g, pr->dtype)) {
    if (int rc = tc4_copy_tables(w.idx, w.wt, st)) return rc;
  } else if (int rc = simt_build_table(g.p, g.d, g.D, w.idx, w.wt, st)) {
    return rc;
  }
  return simt_forward(g, pr->dtype, q, k, v, log_g, y, rowsum, w, st);
}

int pa_power_full_bwd(const pa_problem* pr, const void* q, const void* k, const void* v,
                      const float* log_g, const void* y, const float* rowsum, const void* dy,
                      void* dq, void* dk, void* dv, float* dlog_g, const void* fwd_ws, void* bwd_ws,
                      size_t bwd_ws_bytes, pa_stream_t stream) {
  Geo g;
  if (int rc = make_geo(pr, &g)) return rc;
  if (!q || !k || !v || !y || !dy || !dq || !dk || !dv || !fwd_ws || !bwd_ws ||
      (g.normalize && !rowsum)) {
    set_error("null tensor pointer");
    return PA_ERR_INVALID_SPEC;
  }
  if (!g.gated) dlog_g = nullptr;
  cudaStream_t st = (cudaStream_t)stream;
  bool tc, stage;
  if (int rc = route(pr, g, &tc, &stage)) return rc;
  if (tc && stage) {
    size_t extra;
    PadFwd pf = carve_pad_fwd(g, (char*)fwd_ws + inner_fwd_bytes(g), &extra);
    PadBwd pb = carve_pad_bwd(g, (char*)bwd_ws + inner_bwd_bytes(g), &extra);
    if (bwd_ws_bytes < inner_bwd_bytes(g) + extra) {
      set_error("backward workspace too small");
      return PA_ERR_WORKSPACE;
    }
    stage_in(pb.dy, dy, g, pr->dtype, st);
    if (int rc = tc_backward(g, pf.q, pf.k, pf.v, g.gated ? pf.lg : nullptr, pf.y, g.normalize ? pf.rs : nullptr,
                             pb.dy, pb.dq, pb.dk, pb.dv, dlog_g ? pb.dlg : nullptr, fwd_ws, bwd_ws, st))
      return rc;
    stage_out(dq, pb.dq, g, pr->dtype, st);
    stage_out(dk, pb.dk, g, pr->dtype, st);
    stage_out(dv, pb.dv, g, pr->dtype, st);
    if (dlog_g) unpad_rows(dlog_g, pb.dlg, g, 4, st);
    return cuda_check("padded backward");
  }
  if (tc) {
    if (bwd_ws_bytes < tc_bwd_workspace_bytes(g)) {
      set_error("backward workspace too small");
      return PA_ERR_WORKSPACE;
    }
    return tc_backward(g, q, k, v, log_g, y, rowsum, dy, dq, dk, dv, dlog_g, fwd_ws, bwd_ws, st);
  }
  size_t n1, n2;
  SimtWs w = carve_simt_fwd(g, (void*)fwd_ws, &n1);
  SimtBwdWs b = carve_simt_bwd(g, bwd_ws, &n2);
  if (bwd_ws_bytes < n2) {
    set_error("backward workspace too small");
    return PA_ERR_WORKSPACE;
  }
  return simt_backward(g, pr->dtype, q, k, v, y, rowsum, dy, dq, dk, dv, dlog_g, w, b, st);
}

// ---------------------------------------------------------------- sequence parallel
static int make_sp_geo(const pa_problem* pr, const pa_sp_part* sp, Geo* g) {
  if (int rc = make_geo(pr, g)) return rc;
  if (!sp || sp->chunk0 < 0 || sp->nchunks < g->n || sp->chunk0 + g->n > sp->nchunks) {
    set_error("sequence-parallel partition: need 0 <= chunk0 and chunk0 + local chunks <= nchunks");
    return PA_ERR_INVALID_SPEC;
  }
  if (!tc_supported(*g, pr->dtype) || g->t % g->c) {
    set_error("sequence parallelism runs on the tensor-core path (bf16, p=2, d=e=64, t a multiple of the chunk)");
    return PA_ERR_UNSUPPORTED;
  }
  g->k0 = sp->chunk0;
  g->ng = sp->nchunks;
  g->prefix = sp->chunk0 > 0 ? 1 : 0;
  return PA_OK;
}

size_t pa_sp_state_floats(const pa_problem* pr) {
  return pr ? (size_t)pr->b * pr->h * kSpStateFloatsPerStream : 0;
}

int pa_sp_fwd_local(const pa_problem* pr, const pa_sp_part* sp, const void* q, const void* k, const void* v,
                    const float* log_g, void* ws, size_t ws_bytes, float* end_state, pa_stream_t stream) {
  Geo g;
  if (int rc = make_sp_geo(pr, sp, &g)) return rc;
  if (!q || !k || !v || !ws || !end_state || (g.gated && !log_g)) {
    set_error("null tensor pointer");
    return PA_ERR_INVALID_SPEC;
  }
  if (ws_bytes < tc_fwd_workspace_bytes(g)) {
    set_error("forward workspace too small");
    return PA_ERR_WORKSPACE;
  }
  return tc_forward(g, q, k, v, log_g, nullptr, nullptr, ws, (cudaStream_t)stream, 1, nullptr, end_state);
}

int pa_sp_fwd_finish(const pa_problem* pr, const pa_sp_part* sp, const void* q, const void* k, const void* v,
                     const float* log_g, void* y, float* rowsum, void* ws, size_t ws_bytes, const float* carry,
                     pa_stream_t stream) {
  Geo g;
  if (int rc = make_sp_geo(pr, sp, &g)) return rc;
  if (!q || !k || !v || !y || !ws || (g.gated && !log_g) || (g.prefix && !carry)) {
    set_error("null tensor pointer (a partition after the first needs the incoming state)");
    return PA_ERR_INVALID_SPEC;
  }
  if (ws_bytes < tc_fwd_workspace_bytes(g)) {
    set_error("forward workspace too small");
    return PA_ERR_WORKSPACE;
  }
  return tc_forward(g, q, k, v, log_g, y, rowsum, ws, (cudaStream_t)stream, 2, g.prefix ? carry : nullptr, nullptr);
}

int pa_sp_bwd_local(const pa_problem* pr, const pa_sp_part* sp, const void* q, const void* k, const void* v,
                    const float* log_g, const void* y, const float* rowsum, const void* dy, const void* fwd_ws,
                    void* bwd_ws, size_t bwd_ws_bytes, float* prefix_cot, pa_stream_t stream) {
  Geo g;
  if (int rc = make_sp_geo(pr, sp, &g)) return rc;
  if (!q || !k || !v || !dy || !fwd_ws || !bwd_ws || !prefix_cot || (g.normalize && !rowsum)) {
    set_error("null tensor pointer");
    return PA_ERR_INVALID_SPEC;
  }
  if (bwd_ws_bytes < tc_bwd_workspace_bytes(g)) {
    set_error("backward workspace too small");
    return PA_ERR_WORKSPACE;
  }
  return tc_backward(g, q, k, v, log_g, y, rowsum, dy, nullptr, nullptr, nullptr, nullptr, fwd_ws, bwd_ws,
                     (cudaStream_t)stream, 1, nullptr, prefix_cot);
}

int pa_sp_bwd_finish(const pa_problem* pr, const pa_sp_part* sp, const void* q, const void* k, const void* v,
                     const float* log_g, const void* y, const float* rowsum, const void* dy, void* dq, void* dk,
                     void* dv, float* dlog_g, const void* fwd_ws, void* bwd_ws, size_t bwd_ws_bytes,
                     const float* carry_cot, pa_stream_t stream) {
  Geo g;
  if (int rc = make_sp_geo(pr, sp, &g)) return rc;
  if (!q || !k || !v || !dy || !dq || !dk || !dv || !fwd_ws || !bwd_ws || (g.normalize && !rowsum)) {
    set_error("null tensor pointer");
    return PA_ERR_INVALID_SPEC;
  }
  if (bwd_ws_bytes < tc_bwd_workspace_bytes(g)) {
    set_error("backward workspace too small");
    return PA_ERR_WORKSPACE;
  }
  if (!g.gated) dlog_g = nullptr;
  return tc_backward(g, q, k, v, log_g, y, rowsum, dy, dq, dk, dv, dlog_g, fwd_ws, bwd_ws, (cudaStream_t)stream, 2,
                     carry_cot, nullptr);
}

int pa_sp_combine(const pa_problem* pr, const pa_sp_part* sp, const void* fwd_ws, const float* carry,
                  const float* local, float* out, pa_stream_t stream) {
  Geo g;
  if (int rc = make_sp_geo(pr, sp, &g)) return rc;
  if (!fwd_ws || !local || !out) {
    set_error("null tensor pointer");
    return PA_ERR_INVALID_SPEC;
  }
  return tc_sp_combine(g, fwd_ws, carry, local, out, (cudaStream_t)stream);
}

int pa_fwd_zero_denominators(const pa_problem* pr, const void* ws, pa_stream_t stream,
                             int32_t* count) {
  Geo g;
  if (int rc = make_geo(pr, &g)) return rc;
  // both workspace layouts keep the flag in the first 4 bytes
  cudaError_t e = cudaMemcpyAsync(count, ws, sizeof(int32_t), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) {
    set_error(cudaGetErrorString(e));
    return PA_ERR_CUDA;
  }
  return PA_OK;
}

static int check_op(int n, int c, int d, int e, int p, int dtype) {
  if (n < 1 || c < 1 || d < 1 || e < 1) {
    set_error("need n, c, d, e >= 1");
    return PA_ERR_SHAPE;
  }
  if (p < 1 || p > 4) {
    set_error("power degree p must be in [1, 4] on the CUDA path");
    return PA_ERR_UNSUPPORTED;
  }
  if (dtype != PA_F32 && dtype != PA_F64) {
    set_error("per-operator kernels take f32 or f64");
    return PA_ERR_UNSUPPORTED;
  }
  return PA_OK;
}

// The SPOW per-operator entry points keep one device copy of the monomial
// table per (p, d, device), built on the host and copied synchronously before
// it is published, so no stream can read a half-built table.  They are
// reference-compatibility shims, not the hot path.
static int op_table(int p, int d, const int** idx, const double** wt) {
  struct Ent {
    int* idx;
    double* wt;
  };
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, Ent> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return cuda_check("cudaGetDevice");
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({p, d, dev});
  if (it == cache.end()) {
    const int64_t D = host_binom(d + p - 1, p);
    std::vector<int> hi((size_t)D * p);
    std::vector<double> hw((size_t)D);
    host_feature_table(p, d, hi.data(), hw.data());
    Ent e{nullptr, nullptr};
    if (cudaMalloc(&e.idx, sizeof(int) * hi.size()) != cudaSuccess ||
        cudaMalloc(&e.wt, sizeof(double) * hw.size()) != cudaSuccess ||
        cudaMemcpy(e.idx, hi.data(), sizeof(int) * hi.size(), cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(e.wt, hw.data(), sizeof(double) * hw.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(e.idx);
      cudaFree(e.wt);
      return cuda_check("feature table upload");
    }
    it = cache.emplace(std::make_tuple(p, d, dev), e).first;
  }
  *idx = it->second.idx;
  *wt = it->second.wt;
  return PA_OK;
}

int pa_update_state(int32_t n, int32_t c, int32_t d, int32_t e, int32_t p, int32_t dtype,
                    const void* k, const void* v, const void* w, void* state, void* key_sum,
                    int32_t accumulate, pa_stream_t stream) {
  if (int rc = check_op(n, c, d, e, p, dtype)) return rc;
  const int* idx;
  const double* wt;
  if (int rc = op_table(p, d, &idx, &wt)) return rc;
  int D = (int)host_binom(d + p - 1, p);
  return pub_update(n, c, d, e, p, D, dtype, k, v, w, idx, wt, state, key_sum, accumulate, (cudaStream_t)stream);
}

int pa_query_state(int32_t n, int32_t c, int32_t d, int32_t e, int32_t p, int32_t dtype,
                   const void* q, const void* state, const void* key_sum, void* y, void* denom,
                   int32_t accumulate, pa_stream_t stream) {
  if (int rc = check_op(n, c, d, e, p, dtype)) return rc;
  const int* idx;
  const double* wt;
  if (int rc = op_table(p, d, &idx, &wt)) return rc;
  int D = (int)host_binom(d + p - 1, p);
  return pub_query(n, c, d, e, p, D, dtype, q, state, key_sum, idx, wt, y, denom, accumulate, (cudaStream_t)stream);
}

int64_t pa_expansion_dim(int32_t kind, int32_t p, int32_t d, int32_t d_tile) {
  if (p < 1 || d < 1 || kind < 0 || kind > 2) return -1;
  if (kind == PA_TSPOW && (d_tile < 1 || d % d_tile)) return -1;
  return host_expansion_dim(kind, p, d, d_tile);
}

int pa_expansion_table(int32_t kind, int32_t p, int32_t d, int32_t d_tile, int32_t* idx, double* w) {
  if (pa_expansion_dim(kind, p, d, d_tile) < 0 || p > 4 || !idx || !w) {
    set_error("expansion table needs kind in {spow, tpow, tspow}, 1 <= p <= 4, d >= 1, d_tile | d");
    return PA_ERR_INVALID_SPEC;
  }
  host_expansion_table(kind, p, d, d_tile, idx, w);
  return PA_OK;
}

static int check_table_op(int n, int c, int d, int e, int p, int64_t D, int dtype, const void* idx,
                          const void* wt) {
  if (int rc = check_op(n, c, d, e, p, dtype)) return rc;
  if (D < 1 || D > ((int64_t)1 << 30) || !idx || !wt) {
    set_error("monomial table: need 1 <= D <= 2^30 and device idx / weights");
    return PA_ERR_INVALID_SPEC;
  }
  return PA_OK;
}

int pa_update_state_table(int32_t n, int32_t c, int32_t d, int32_t e, int32_t p, int64_t D, int32_t dtype,
                          const void* k, const void* v, const void* w, const int32_t* idx, const double* weights,
                          void* state, void* key_sum, int32_t accumulate, pa_stream_t stream) {
  if (int rc = check_table_op(n, c, d, e, p, D, dtype, idx, weights)) return rc;
  return pub_update(n, c, d, e, p, (int)D, dtype, k, v, w, idx, weights, state, key_sum, accumulate,
                    (cudaStream_t)stream);
}

int pa_query_state_table(int32_t n, int32_t c, int32_t d, int32_t e, int32_t p, int64_t D, int32_t dtype,
                         const void* q, const void* state, const void* key_sum, const int32_t* idx,
                         const double* weights, void* y, void* denom, int32_t accumulate, pa_stream_t stream) {
  if (int rc = check_table_op(n, c, d, e, p, D, dtype, idx, weights)) return rc;
  return pub_query(n, c, d, e, p, (int)D, dtype, q, state, key_sum, idx, weights, y, denom, accumulate,
                   (cudaStream_t)stream);
}

int pa_discumsum(int32_t n, int64_t L, int64_t M, int32_t dtype, const void* values,
                 const void* lams, void* out, pa_stream_t stream) {
  if (n < 1 || L < 1 || M < 1) {
    set_error("need n, L, M >= 1");
    return PA_ERR_SHAPE;
  }
  if (dtype != PA_F32 && dtype != PA_F64) {
    set_error("discumsum takes f32 or f64");
    return PA_ERR_UNSUPPORTED;
  }
  return pub_discumsum(n, L, M, dtype, values, lams, out, (cudaStream_t)stream);
}

int pa_profile_enable(int32_t on) {
  if (!on) prof_drain();
  g_prof_on.store(on != 0);
  return PA_OK;
}

void pa_profile_reset(void) {
  prof_drain();
  std::lock_guard<std::mutex> lk(g_pm);
  g_prof_acc.clear();
}

int pa_profile_read(char* names, double* ms, int64_t* launches, int32_t cap) {
  prof_drain();
  std::lock_guard<std::mutex> lk(g_pm);
  int i = 0;
  for (auto& kv : g_prof_acc) {
    if (i >= cap) break;
    strncpy(names + 32 * i, kv.first.c_str(), 31);
    names[32 * i + 31] = 0;
    ms[i] = kv.second.first;
    launches[i] = kv.second.second;
    ++i;
  }
  return i;
}

const char* pa_last_error(void) { return g_err.c_str(); }
int64_t pa_launch_count(void) { return g_launches.load(); }

}  // extern "C"
