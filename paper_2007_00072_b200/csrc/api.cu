// C ABI of libencoder.so (include/encoder.h): argument validation, the enc_ctx, buffer
// layouts, and the encoder-layer forward/backward orchestration (operator order of Table
// A.1).  Everything runs on `stream`; nothing synchronises.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <climits>

#include <atomic>
#include <mutex>
#include <new>
#include <unordered_map>

#include "../../include/encoder.h"
#include "gemm.h"
#include "kernels.h"

using namespace enc;

// ENC_OPT_PDL (process-wide: the launch helpers have no context): programmatic dependent
// launch of the kernels that call pdl_wait() (kernels.h launch_k)
static constexpr int kPdlDefault = PDL_LN | PDL_ATTN_BH | PDL_WGEMM;   // measured at L (DESIGN 8.6)
static std::atomic<int> g_pdl{-1};
bool enc::pdl_enabled(int cls) {
  int v = g_pdl.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = getenv("ENC_PDL");
    v = e ? (int)strtol(e, nullptr, 0) : kPdlDefault;
    g_pdl.store(v, std::memory_order_relaxed);
  }
  return (v & cls) != 0;
}
void enc::pdl_set(int mask) { g_pdl.store(mask, std::memory_order_relaxed); }

struct enc_ctx {
  int device = 0;
  int num_sms = 148;
  cublasHandle_t blas = nullptr;
  void* blas_ws = nullptr;
  size_t blas_ws_bytes = 0;
  float* red = nullptr;      // column-reduction partials
  size_t red_floats = 0;
  // optional per-operator CUDA-event timing (enc_set_timing / enc_op_times)
  uint64_t timing_mask = 0;
  cudaEvent_t ev0[ENC_NUM_OPS] = {};
  cudaEvent_t ev1[ENC_NUM_OPS] = {};
  bool recorded[ENC_NUM_OPS] = {};
  uint64_t launches = 0;     // kernels this library launched (excluding cuBLAS)
  int attn_tc = 1;           // ENC_OPT_ATTN_TC
  int attn_fused = 1;        // ENC_OPT_ATTN_FUSED
  int attn_bh = 1;           // ENC_OPT_ATTN_BH
  int qkv_direct = 1;        // ENC_OPT_QKV_DIRECT
  LtCtx* lt = nullptr;       // cuBLASLt + measured algorithm cache (weight GEMMs)
  int use_lt = 1;            // ENC_OPT_GEMM_LT
  // encoder_layer_step_host: host<->device copies on their own streams, overlapped with
  // the layer (dY in during the forward, Y out during the backward)
  cudaStream_t copy_in = nullptr, copy_out = nullptr;
  cudaEvent_t ev_in = nullptr, ev_fwd = nullptr, ev_out = nullptr, ev_start = nullptr;
  // backward: weight-gradient contractions on a side stream (own cuBLASLt workspace),
  // forked after their inputs are ready and joined at the end of each backward part
  int bwd_side = 3;          // ENC_OPT_BWD_SIDE (3: finalize beside the last contractions;
                             // GEMMs on a side stream measured slower with PDL)
  int attn_overlap = 0;      // ENC_OPT_ATTN_OVERLAP: dV beside the fused dA + BSB-bwd (off:
                             // -7 us per step, but the fused kernel's own time then includes
                             // the SMs it shares with dV)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // the backward's column-sum finalize beside the last weight contractions
  cudaStream_t side2 = nullptr;
  cudaEvent_t ev_fork2 = nullptr, ev_join2 = nullptr;
  // the FFN keep bytes drawn ahead beside the fused score kernel (R29)
  cudaEvent_t ev_mk_fork = nullptr, ev_mk_join = nullptr;
  int mask_ahead = 1;      // ENC_OPT_MASK_AHEAD (FFN bytes on the fused kernel's spare SMs, R31)
  // ENC_OPT_SIDE_OPS (dW contractions on the side stream): Out-dW beside the fused BSB-bwd /
  // dQdK stretch (measured -2..-6 us at L); the others measured neutral or slower
  uint32_t side_ops = 1u << ENC_OP_GEMM_OUT_DW;
  int attn_fused_av = 1;   // ENC_OPT_ATTN_FUSED_AV (QK^T + BSB + A.V in one kernel, R30)
  void* side_ws = nullptr;
  // pipelined host steps: input copies done (ev_pf, on copy_in), fork point on the layer
  // stream (ev_pfs)
  cudaEvent_t ev_pf = nullptr, ev_pfs = nullptr, ev_bwd = nullptr;
  // fused forward: the attention keep words generated on the side stream beside the QKV
  // contraction (ENC_OPT_KEEP_AHEAD), joined before the score kernel
  int keep_ahead = 0;
  int qkv_fusion = ENC_QKV_STACKED;   // ENC_OPT_QKV_FUSION (Table A.2 algebraic fusion)
  int qkv_fusion_bwd = ENC_QKV_STACKED;   // its backward dX / dW grouping
  int bdrln_variant = 0;   // ENC_OPT_BDRLN_VARIANT (kernel / warps per row of BDRLN, -bwd)
  int attn_dc = 1;         // ENC_OPT_ATTN_DC (fused BSB-bwd row term from C, R26)
  int mask_bytes = 1;      // ENC_OPT_MASK_BYTES (BDRLN / BAD keep bytes stored, R27)
  int av_keep_gen = 0;     // ENC_OPT_AV_KEEP_GEN (attention keep words generated in A.V, R28;
                           // measured +4 us at L: off)
  cudaEvent_t ev_kb_fork = nullptr, ev_kb_join = nullptr;
  // hand-written tcgen05 weight contractions (wgemm.cu) for bf16: ENC_OPT_GEMM_TC
  // weight contractions on the tcgen05 kernel: bit (1 << ENC_OP_GEMM_*) per contraction.
  // Default = the measured selection at configs L and Bb: the two
  // fused FFN kernels (Linear1 + BAD, Linear2-dX + BAD-bwd) on tcgen05, the plain
  // contractions on cuBLASLt (its tuned kernels measured 2-8 us faster per contraction)
  uint32_t gemm_tc = (1u << ENC_OP_GEMM_L1) | (1u << ENC_OP_GEMM_L2_DX);
  int gemm_cg = 0;           // ENC_OPT_GEMM_PAIR 1 (default) -> 0 (auto), 0 -> 1 (single CTAs)
  void* wg_ws = nullptr;     // split-K partial slabs of the fp32 weight-gradient outputs
  void* wg_ws_side = nullptr;   // the same for contractions on the side stream
  size_t wg_ws_bytes = 0;
  // forward -> backward contract: the path flags each `saved` buffer was written with
  std::mutex mu;
  std::unordered_map<const void*, uint32_t> saved_paths;
};

// Weight contraction: row-major C[M,N] = op(A) op(B) (+ beta C), nn.Linear operand layouts
// (tA: A stored [K][M]; tB: B stored [N][K]).  bf16: the hand-written tcgen05 kernel
// (wgemm.cu) with an optional fp32 bias over columns; fp32 (or ENC_OPT_GEMM_TC off):
// cuBLASLt / cuBLAS.  Returns an ENC_* code.
static int wcontract(enc_ctx* ctx, int op, cudaStream_t st, int in_dt, int out_dt, bool tA,
                     bool tB, int M, int N, int K, const void* A, int lda, const void* B,
                     int ldb, float beta, void* C, int ldc, const float* bias = nullptr,
                     void* lt_ws = nullptr);

// Groups of stacked Q / K / V weight blocks (block 0 = Q, 1 = K, 2 = V) contracted together
// under each algebraic-fusion variant of Table A.2
static void qkv_groups(int mode, int* n, int* start, int* count) {
  switch (mode) {
    case ENC_QKV_SEPARATE: *n = 3; start[0] = 0; start[1] = 1; start[2] = 2;
      count[0] = count[1] = count[2] = 1; return;
    case ENC_QKV_QK_STACKED: *n = 2; start[0] = 0; count[0] = 2; start[1] = 2; count[1] = 1;
      return;
    case ENC_QKV_KV_STACKED: *n = 2; start[0] = 0; count[0] = 1; start[1] = 1; count[1] = 2;
      return;
    default: *n = 1; start[0] = 0; count[0] = 3; return;
  }
}

// weight contractions: cuBLASLt with per-shape measured algorithm choice, or cuBLAS
static cublasStatus_t wgemm(enc_ctx* ctx, cudaStream_t st, int in_dt, int out_dt, bool tA,
                            bool tB, int M, int N, int K, float alpha, const void* A, int lda,
                            const void* B, int ldb, float beta, void* C, int ldc,
                            void* ws = nullptr) {
  if (ctx->lt && ctx->use_lt && alpha == 1.f)
    return lt_gemm_rm(ctx->lt, in_dt, out_dt, tA, tB, M, N, K, A, lda, B, ldb, beta, C, ldc,
                      LT_EPI_NONE, nullptr, st, ws);
  return gemm_rm(ctx->blas, in_dt, out_dt, tA, tB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc);
}

// Same with a cuBLASLt epilogue (LT_EPI_BIAS / LT_EPI_BGRAD_A into `bias`).  Returns false
// (nothing launched) when the epilogue is unavailable -- cuBLAS path selected, or no
// cuBLASLt algorithm for it -- and the caller then runs the plain contraction plus its own
// bias kernel.
static bool wgemm_epi(enc_ctx* ctx, cudaStream_t st, int in_dt, int out_dt, bool tA, bool tB,
                      int M, int N, int K, const void* A, int lda, const void* B, int ldb,
                      void* C, int ldc, int epi, float* bias) {
  if (!ctx->lt || !ctx->use_lt) return false;
  return lt_gemm_rm(ctx->lt, in_dt, out_dt, tA, tB, M, N, K, A, lda, B, ldb, 0.f, C, ldc, epi,
                    bias, st) == CUBLAS_STATUS_SUCCESS;
}

namespace {
const char* kOpNames[ENC_NUM_OPS] = {
    "gemm_qkv", "aib_fwd", "gemm_qk", "bsb_fwd", "gemm_av", "gemm_out", "bdrln_fwd1",
    "gemm_l1", "bad_fwd", "gemm_l2", "bdrln_fwd2", "bdrln_bwd2", "gemm_l2_dx", "gemm_l2_dw",
    "bad_bwd", "gemm_l1_dx", "gemm_l1_dw", "bdrln_bwd1", "gemm_out_dx", "gemm_out_dw",
    "gemm_av_da", "gemm_av_dv", "bsb_bwd", "gemm_qk_dq", "gemm_qk_dk", "aib_bwd",
    "gemm_qkv_dx", "gemm_qkv_dw"};

// Records CUDA events around one operator on `st` when its bit is set in timing_mask.
struct OpTimer {
  enc_ctx* c;
  int op;
  cudaStream_t st;
  bool on;
  // active = false: the operator is fused into another kernel on this path (no work of its
  // own, not timed: enc_op_times reports -1 for it)
  OpTimer(enc_ctx* c_, int op_, cudaStream_t st_, int launches, bool active = true)
      : c(c_), op(op_), st(st_), on(active && ((c_->timing_mask >> op_) & 1ull)) {
    c->launches += launches;
    if (on) record(c->ev0[op]);
  }
  ~OpTimer() {
    if (on) {
      record(c->ev1[op]);
      c->recorded[op] = true;
    }
  }
  // inside CUDA-graph capture the event must become an event-record node of the graph
  void record(cudaEvent_t ev) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(st, &cs);
    if (cs == cudaStreamCaptureStatusActive)
      cudaEventRecordWithFlags(ev, st, cudaEventRecordExternal);
    else
      cudaEventRecord(ev, st);
  }
};
}  // namespace

static thread_local int g_last_cuda = 0;

static int cuda_fail(cudaError_t e) {
  g_last_cuda = (int)e;
  return ENC_ECUDA;
}
#define CK(x)                                  \
  do {                                         \
    cudaError_t _e = (x);                      \
    if (_e != cudaSuccess) return cuda_fail(_e); \
  } while (0)
#define CB(x)                                           \
  do {                                                  \
    cublasStatus_t _s = (x);                            \
    if (_s != CUBLAS_STATUS_SUCCESS) return ENC_ECUBLAS; \
  } while (0)

static int wcontract(enc_ctx* ctx, int op, cudaStream_t st, int in_dt, int out_dt, bool tA,
                     bool tB, int M, int N, int K, const void* A, int lda, const void* B,
                     int ldb, float beta, void* C, int ldc, const float* bias, void* lt_ws) {
  if (((ctx->gemm_tc >> op) & 1u) && in_dt == ENC_BF16 && (beta == 0.f || beta == 1.f)) {
    WgemmArgs g;
    g.M = M; g.N = N; g.K = K;
    g.A = A; g.lda = lda; g.a_mn = tA ? 1 : 0;
    g.B = B; g.ldb = ldb; g.b_mn = tB ? 0 : 1;
    g.C = C; g.ldc = ldc; g.out_f32 = out_dt == ENC_FP32 ? 1 : 0;
    g.beta = beta != 0.f ? 1 : 0;
    g.bias = bias;
    g.ws = lt_ws ? ctx->wg_ws_side : ctx->wg_ws;   // lt_ws set: the side stream's call
    g.ws_bytes = ctx->wg_ws_bytes;
    g.cg = ctx->gemm_cg;
    if (wgemm_supported(g)) {
      const cudaError_t e = launch_wgemm(g, ctx->num_sms, st);
      if (e != cudaSuccess) return cuda_fail(e);
      ctx->launches += wgemm_launches(g, ctx->num_sms);
      return ENC_OK;
    }
  }
  if (bias) {
    if (out_dt == ENC_FP32 || in_dt != ENC_BF16) {
      // fp32 output: cuBLASLt takes the fp32 bias directly
      if (ctx->lt && ctx->use_lt && beta == 0.f &&
          lt_gemm_rm(ctx->lt, in_dt, out_dt, tA, tB, M, N, K, A, lda, B, ldb, 0.f, C, ldc,
                     LT_EPI_BIAS, const_cast<float*>(bias), st) == CUBLAS_STATUS_SUCCESS)
        return ENC_OK;
    }
    return ENC_EUNSUPPORTED;   // the caller adds the bias itself
  }
  return wgemm(ctx, st, in_dt, out_dt, tA, tB, M, N, K, 1.f, A, lda, B, ldb, beta, C, ldc, lt_ws)
             == CUBLAS_STATUS_SUCCESS
             ? ENC_OK
             : ENC_ECUBLAS;
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }
static size_t esize(int dtype) { return dtype == ENC_BF16 ? 2 : 4; }
static bool valid_dtype(int dtype) { return dtype == ENC_BF16 || dtype == ENC_FP32; }
// p in [0, 1) whose 16-bit threshold T = floor(65536 p + 1/2) (R5) is below 65536:
// p >= 1 - 2^-17 would give T = 65536, i.e. no kept value and an infinite scale
static bool valid_p(float p) {
  return p >= 0.f && p < 1.f && p == p && floor((double)p * 65536.0 + 0.5) < 65536.0;
}

extern "C" {

const char* enc_strerror(int code) {
  switch (code) {
    case ENC_OK: return "ok";
    case ENC_EINVAL: return "invalid argument (dimension, p, or K != J / W != P / I != H*P)";
    case ENC_EALIGN: return "misaligned pointer (16 B) or dimension not a multiple of 8";
    case ENC_EDTYPE: return "unknown dtype";
    case ENC_ECUDA: return "CUDA error (see enc_last_cuda_error)";
    case ENC_ECUBLAS: return "cuBLAS error";
    case ENC_EUNSUPPORTED: return "shape outside the compiled kernel variants";
    case ENC_ENULL: return "required pointer is NULL";
    default: return "unknown error";
  }
}

int enc_last_cuda_error(void) { return g_last_cuda; }

const char* enc_version(void) { return "paper_2007_00072_b200 0.1 sm_100a"; }

int enc_create(enc_ctx** out, int device) {
  if (!out) return ENC_ENULL;
  *out = nullptr;
  int prev = 0;
  CK(cudaGetDevice(&prev));
  CK(cudaSetDevice(device));
  enc_ctx* c = new (std::nothrow) enc_ctx();
  if (!c) return ENC_EINVAL;
  c->device = device;
  cudaError_t e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) { delete c; cudaSetDevice(prev); return cuda_fail(e); }
  if (cublasCreate(&c->blas) != CUBLAS_STATUS_SUCCESS) { delete c; cudaSetDevice(prev); return ENC_ECUBLAS; }
  c->blas_ws_bytes = 32u << 20;
  c->red_floats = (64u << 20) / sizeof(float);
  e = cudaMalloc(&c->blas_ws, c->blas_ws_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->red, c->red_floats * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&c->side_ws, c->blas_ws_bytes);
  c->wg_ws_bytes = 32u << 20;
  if (e == cudaSuccess) e = cudaMalloc(&c->wg_ws, c->wg_ws_bytes);
  if (e == cudaSuccess) e = cudaMalloc(&c->wg_ws_side, c->wg_ws_bytes);
  if (e != cudaSuccess) { enc_destroy(c); cudaSetDevice(prev); return cuda_fail(e); }
  if (cublasSetWorkspace(c->blas, c->blas_ws, c->blas_ws_bytes) != CUBLAS_STATUS_SUCCESS ||
      cublasSetMathMode(c->blas, CUBLAS_DEFAULT_MATH) != CUBLAS_STATUS_SUCCESS) {
    enc_destroy(c);
    cudaSetDevice(prev);
    return ENC_ECUBLAS;
  }
  for (int i = 0; i < ENC_NUM_OPS && e == cudaSuccess; ++i) {
    e = cudaEventCreate(&c->ev0[i]);
    if (e == cudaSuccess) e = cudaEventCreate(&c->ev1[i]);
  }
  if (e != cudaSuccess) { enc_destroy(c); cudaSetDevice(prev); return cuda_fail(e); }
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy_in, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->side2, cudaStreamNonBlocking);
  cudaEvent_t* evs[15] = {&c->ev_in,   &c->ev_fwd, &c->ev_out, &c->ev_start,
                          &c->ev_fork, &c->ev_join, &c->ev_pf,  &c->ev_pfs,
                          &c->ev_bwd,  &c->ev_kb_fork, &c->ev_kb_join, &c->ev_fork2,
                          &c->ev_join2, &c->ev_mk_fork, &c->ev_mk_join};
  for (int i = 0; i < 15 && e == cudaSuccess; ++i)
    e = cudaEventCreateWithFlags(evs[i], cudaEventDisableTiming);
  if (e != cudaSuccess) { enc_destroy(c); cudaSetDevice(prev); return cuda_fail(e); }
  c->lt = lt_create(c->blas_ws, c->blas_ws_bytes);  // optional: cuBLAS is the fallback
  cudaSetDevice(prev);
  *out = c;
  return ENC_OK;
}

int enc_num_ops(void) { return ENC_NUM_OPS; }

const char* enc_op_name(int op) { return (op >= 0 && op < ENC_NUM_OPS) ? kOpNames[op] : ""; }

int enc_set_timing(enc_ctx* c, uint64_t op_mask) {
  if (!c) return ENC_ENULL;
  c->timing_mask = op_mask;
  for (int i = 0; i < ENC_NUM_OPS; ++i) c->recorded[i] = false;
  return ENC_OK;
}

int enc_op_times(enc_ctx* c, float* ms) {
  if (!c || !ms) return ENC_ENULL;
  for (int i = 0; i < ENC_NUM_OPS; ++i) {
    ms[i] = -1.f;
    if (!c->recorded[i]) continue;
    CK(cudaEventSynchronize(c->ev1[i]));
    CK(cudaEventElapsedTime(&ms[i], c->ev0[i], c->ev1[i]));
  }
  return ENC_OK;
}

uint64_t enc_launch_count(const enc_ctx* c) { return c ? c->launches : 0; }

void enc_destroy(enc_ctx* c) {
  if (!c) return;
  for (int i = 0; i < ENC_NUM_OPS; ++i) {
    if (c->ev0[i]) cudaEventDestroy(c->ev0[i]);
    if (c->ev1[i]) cudaEventDestroy(c->ev1[i]);
  }
  if (c->lt) lt_destroy(c->lt);
  for (cudaEvent_t ev : {c->ev_in, c->ev_fwd, c->ev_out, c->ev_start, c->ev_fork, c->ev_join,
                         c->ev_pf, c->ev_pfs, c->ev_bwd, c->ev_kb_fork, c->ev_kb_join,
                         c->ev_fork2, c->ev_join2, c->ev_mk_fork, c->ev_mk_join})
    if (ev) cudaEventDestroy(ev);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->side2) cudaStreamDestroy(c->side2);
  if (c->side_ws) cudaFree(c->side_ws);
  if (c->copy_in) cudaStreamDestroy(c->copy_in);
  if (c->copy_out) cudaStreamDestroy(c->copy_out);
  if (c->blas) cublasDestroy(c->blas);
  if (c->blas_ws) cudaFree(c->blas_ws);
  if (c->red) cudaFree(c->red);
  if (c->wg_ws) cudaFree(c->wg_ws);
  if (c->wg_ws_side) cudaFree(c->wg_ws_side);
  delete c;
}

}  // extern "C"

static ReduceWs ws_of(const enc_ctx* c) { return ReduceWs{c->red, c->red_floats, c->num_sms}; }

// One attention contraction (ENC_AG_*) on the per-(b, h) streaming kernel when it applies,
// else on the tiled tcgen05 kernel.
static bool use_bh(const enc_ctx* ctx, int J, int P) {
  return ctx->attn_bh && attn_bh_supported(J, P);
}
static bool tc_attn_of(const enc_ctx* ctx, int dtype, int J, int P) {
  return ctx->attn_tc && dtype == ENC_BF16 && attn_gemm_supported(J, P);
}
static cudaError_t attn_contract(const enc_ctx* ctx, int which, int B, int H, int J, int P,
                                 const void* X, int64_t ldx, const void* Y, int64_t ldy, void* Z,
                                 int64_t ldz, cudaStream_t st) {
  if (use_bh(ctx, J, P)) {
    switch (which) {
      case ENC_AG_AV: return launch_attn_av_bh(B, H, J, P, X, Y, ldy, Z, ldz, nullptr, 1.f, st);
      case ENC_AG_DV:
        return launch_attn_dv_bh(B, H, J, P, X, Y, ldy, Z, ldz, nullptr, 0, nullptr, 1.f, st);
      case ENC_AG_DQ:
        return launch_attn_dqdk_bh(B, H, J, P, X, Y, ldy, nullptr, 0, Z, ldz, nullptr, 0,
                                   nullptr, nullptr, 0, st);
      case ENC_AG_DK:
        return launch_attn_dqdk_bh(B, H, J, P, X, nullptr, 0, Y, ldy, nullptr, 0, Z, ldz,
                                   nullptr, nullptr, 0, st);
      default: break;
    }
  }
  return launch_attn_gemm(which, B, H, J, P, X, ldx, Y, ldy, Z, ldz, st);
}

// ------------------------------------------------------------------ dims validation
static int check_dims(const enc_dims* d, int dtype) {
  if (!d) return ENC_ENULL;
  if (!valid_dtype(dtype)) return ENC_EDTYPE;
  if (d->B < 0 || d->J <= 0 || d->H <= 0 || d->P <= 0 || d->U <= 0) return ENC_EINVAL;
  if (d->K != d->J || d->W != d->P || d->I != d->H * d->P) return ENC_EINVAL;
  if (d->I % 8 || d->U % 8 || d->K % 8 || d->P % 8) return ENC_EALIGN;
  if (!rowop_supported(d->K) || !rowop_supported(d->I)) return ENC_EUNSUPPORTED;
  if (!bdrln_bwd_supported(d->I, dtype)) return ENC_EUNSUPPORTED;
  // chunk / row indices are 32-bit inside the kernels
  const int64_t wide = 3 * d->I > d->U ? 3 * d->I : d->U;
  if ((int64_t)d->B * d->J * wide / 8 >= INT32_MAX || (int64_t)d->B * d->H * d->J >= INT32_MAX)
    return ENC_EUNSUPPORTED;
  return ENC_OK;
}

static int check_cfg(const enc_cfg* c) {
  if (!c) return ENC_ENULL;
  if (!valid_p(c->p_attn) || !valid_p(c->p_hidden) || !valid_p(c->p_ffn)) return ENC_EINVAL;
  if (c->act < ENC_ACT_GELU_ERF || c->act > ENC_ACT_RELU) return ENC_EINVAL;
  if (!(c->ln_eps >= 0.f)) return ENC_EINVAL;
  if (c->batch_offset < 0) return ENC_EINVAL;
  if (c->causal != 0 && c->causal != 1) return ENC_EINVAL;
  return ENC_OK;
}

#define CHECK_PTRS(...)                                        \
  do {                                                         \
    const void* _ps[] = {__VA_ARGS__};                         \
    for (const void* _p : _ps) {                               \
      if (!_p) return ENC_ENULL;                               \
      if (!aligned16(_p)) return ENC_EALIGN;                   \
    }                                                          \
  } while (0)

// ------------------------------------------------------------------ buffer layouts
namespace {
enum SavedId { S_Q, S_K, S_V, S_P, S_A, S_C, S_X1, S_XH1, S_H, S_A1, S_XH2, S_R1, S_R2, S_KB,
               S_CLO, S_KB1, S_KBF, S_KB2, S_N };
enum FwdId { F_PTR, F_QKV, F_S, F_YO, F_Y2, F_N };
enum BwdId { B_PTR, B_DY2, B_DA1, B_DH, B_DX1, B_DYO, B_DC, B_DA, B_DS, B_DQ, B_DK, B_DV, B_DQKV, B_N };

struct Layout {
  size_t off[20];
  size_t total;
};

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

static Layout make_layout(const size_t* sizes, int n) {
  Layout L;
  size_t o = 0;
  for (int i = 0; i < n; ++i) {
    L.off[i] = o;
    o += al(sizes[i]);
  }
  L.total = o;
  return L;
}

struct Sizes {
  size_t BJI, BJU, BHJK, BJ3I, BJ, ptr, KB, KBI, KBU;
};
static Sizes sizes_of(const enc_dims* d, int dtype) {
  const size_t es = esize(dtype);
  const size_t BJ = (size_t)d->B * d->J;
  Sizes s;
  s.BJI = BJ * d->I * es;
  s.BJU = BJ * d->U * es;
  s.BHJK = (size_t)d->B * d->H * d->J * d->K * es;
  s.BJ3I = BJ * 3 * d->I * es;
  s.BJ = BJ * sizeof(float);
  s.ptr = (size_t)5 * d->B * d->H * sizeof(void*);
  s.KB = (size_t)d->B * d->H * d->J * ((d->K + 31) / 32) * sizeof(uint32_t);  // keep-flag words
  s.KBI = BJ * (size_t)(d->I / 8);   // keep bytes of a hidden-size dropout site (R27)
  s.KBU = BJ * (size_t)(d->U / 8);   // keep bytes of the FFN dropout site
  return s;
}
static Layout saved_layout(const enc_dims* d, int dtype) {
  const Sizes s = sizes_of(d, dtype);
  // S_CLO: the attention output's rounding residual (bf16 path, R26)
  // S_KB1 / S_KBF / S_KB2: keep bytes of BDRLN site 1, BAD, BDRLN site 2 (R27)
  const size_t sz[S_N] = {s.BJI, s.BJI, s.BJI, s.BHJK, s.BHJK, s.BJI, s.BJI, s.BJI,
                          s.BJU, s.BJU, s.BJI, s.BJ,   s.BJ,   s.KB,  s.BJI, s.KBI,
                          s.KBU, s.KBI};
  return make_layout(sz, S_N);
}
static Layout fwd_layout(const enc_dims* d, int dtype) {
  const Sizes s = sizes_of(d, dtype);
  const size_t sz[F_N] = {s.ptr, s.BJ3I, s.BHJK, s.BJI, s.BJI};
  return make_layout(sz, F_N);
}
static Layout bwd_layout(const enc_dims* d, int dtype) {
  const Sizes s = sizes_of(d, dtype);
  const size_t sz[B_N] = {s.ptr, s.BJI,  s.BJU, s.BJU, s.BJI, s.BJI, s.BJI,
                          s.BHJK, s.BHJK, s.BJI, s.BJI, s.BJI, s.BJ3I};
  return make_layout(sz, B_N);
}
static inline char* at(void* base, size_t off) { return (char*)base + off; }
}  // namespace

// Linear1 + BAD (EPI_BAD_FWD) and Linear2-dX + BAD-bwd (EPI_BAD_BWD) on the tcgen05 kernel;
// M = 0 (rejected by wgemm_supported) when that path is off for this call
static WgemmArgs ffn_fwd_args(const enc_ctx* ctx, const enc_dims* d, int dtype,
                              const enc_cfg* cfg, const void* X1, const void* W1, const float* b1,
                              const PhiloxKey& pk, void* h, void* A1, bool force = false) {
  WgemmArgs g;
  if ((!((ctx->gemm_tc >> ENC_OP_GEMM_L1) & 1u) && !force) || dtype != ENC_BF16) return g;
  g.ws = ctx->wg_ws;
  g.ws_bytes = ctx->wg_ws_bytes;
  g.M = d->B * d->J; g.N = d->U; g.K = d->I;
  g.A = X1; g.lda = d->I;
  g.B = W1; g.ldb = d->I;
  g.C = h; g.ldc = d->U;
  g.C2 = A1; g.ldc2 = d->U;
  g.epi = EPI_BAD_FWD;
  g.cg = ctx->gemm_cg;
  g.bias = b1;
  g.act = cfg->act;
  g.pk = pk;
  g.g0 = cfg->batch_offset * (int64_t)d->J * (d->U / 8);
  return g;
}
static WgemmArgs ffn_bwd_args(const enc_ctx* ctx, const enc_dims* d, int dtype,
                              const enc_cfg* cfg, const void* dY2, const void* W2, const void* h,
                              const PhiloxKey& pk, void* dh, float* partials, bool force = false) {
  WgemmArgs g;
  if ((!((ctx->gemm_tc >> ENC_OP_GEMM_L2_DX) & 1u) && !force) || dtype != ENC_BF16) return g;
  g.ws = ctx->wg_ws;
  g.ws_bytes = ctx->wg_ws_bytes;
  g.M = d->B * d->J; g.N = d->U; g.K = d->I;
  g.A = dY2; g.lda = d->I;
  g.B = W2; g.ldb = d->U; g.b_mn = 1;
  g.C = dh; g.ldc = d->U;
  g.aux = h; g.ldaux = d->U;
  g.partials = partials;
  g.epi = EPI_BAD_BWD;
  g.cg = ctx->gemm_cg;
  g.act = cfg->act;
  g.pk = pk;
  g.g0 = cfg->batch_offset * (int64_t)d->J * (d->U / 8);
  return g;
}

extern "C" {

int enc_layer_sizes(const enc_dims* d, int dtype, size_t* saved_bytes, size_t* scratch_bytes) {
  int r = check_dims(d, dtype);
  if (r) return r;
  if (saved_bytes) *saved_bytes = saved_layout(d, dtype).total;
  if (scratch_bytes) {
    const size_t f = fwd_layout(d, dtype).total, b = bwd_layout(d, dtype).total;
    *scratch_bytes = f > b ? f : b;
  }
  return ENC_OK;
}

// The tcgen05 attention paths consume the QKV contraction output in place: Q, K, V are the
// three column blocks of one [B, J, 3I] tensor spanning the Q, K, V regions (row stride 3I),
// and dQ, dK, dV the blocks of dQKV.  Other paths: separate [B,H,J,P] tensors.
static bool qkv_direct(const enc_ctx* ctx, const enc_dims* d, int dtype) {
  return ctx->qkv_direct && tc_attn_of(ctx, dtype, d->J, d->P);
}

// The attention-path flags a forward wrote `saved` with (Q/K/V in place or permuted, fused
// score kernels, A stored or applied on load): the backward must read it the same way
// The fused BSB-bwd takes its row term from C = C_hi + C_lo (R26) when the forward wrote the
// low word: fused score path with A.V on the per-(b,h) kernel, J = K = 512
static bool dc_term_of(const enc_ctx* ctx, bool fused_attn, int J, int P) {
  return fused_attn && use_bh(ctx, J, P) && ctx->attn_dc && !attn_short_supported(J, P);
}

// The forward stores keep bytes (R27) of both BDRLN sites when ENC_OPT_MASK_BYTES is on, and
// of BAD when it also runs in the Linear1 contraction's epilogue
static bool bad_bytes_of(const enc_ctx* ctx, const enc_dims* d, int dtype) {
  return ctx->mask_bytes && dtype == ENC_BF16 && ((ctx->gemm_tc >> ENC_OP_GEMM_L1) & 1u) &&
         d->U % 8 == 0 && d->I % 8 == 0;
}

static uint32_t path_flags(const enc_ctx* ctx, const enc_dims* d, int dtype) {
  const bool tc = tc_attn_of(ctx, dtype, d->J, d->P);
  const bool fused = tc && ctx->attn_fused && attn_fused_supported(d->J, d->P);
  return (qkv_direct(ctx, d, dtype) ? 1u : 0u) | (tc ? 2u : 0u) | (fused ? 4u : 0u) |
         (fused && use_bh(ctx, d->J, d->P) ? 8u : 0u) |
         (dc_term_of(ctx, fused, d->J, d->P) ? 16u : 0u) | (ctx->mask_bytes ? 32u : 0u) |
         (bad_bytes_of(ctx, d, dtype) ? 64u : 0u) | 0x100u;
}

int enc_saved_views(enc_ctx* ctx, const enc_dims* d, int dtype, void* saved, enc_saved_view* v) {
  if (!ctx) return ENC_ENULL;
  int r = check_dims(d, dtype);
  if (r) return r;
  if (!saved || !v) return ENC_ENULL;
  const Layout L = saved_layout(d, dtype);
  const size_t ies = (size_t)d->I * esize(dtype);
  if (qkv_direct(ctx, d, dtype)) {
    v->Q = at(saved, L.off[S_Q]);
    v->K = at(saved, L.off[S_Q] + ies);
    v->V = at(saved, L.off[S_Q] + 2 * ies);
    v->qkv_ld = 3LL * d->I;
  } else {
    v->Q = at(saved, L.off[S_Q]);
    v->K = at(saved, L.off[S_K]);
    v->V = at(saved, L.off[S_V]);
    v->qkv_ld = d->P;
  }
  v->P = at(saved, L.off[S_P]);
  v->A = at(saved, L.off[S_A]);
  v->C = at(saved, L.off[S_C]);
  v->X1 = at(saved, L.off[S_X1]);
  v->xhat1 = at(saved, L.off[S_XH1]);
  v->h = at(saved, L.off[S_H]);
  v->A1 = at(saved, L.off[S_A1]);
  v->xhat2 = at(saved, L.off[S_XH2]);
  v->rstd1 = (float*)at(saved, L.off[S_R1]);
  v->rstd2 = (float*)at(saved, L.off[S_R2]);
  v->keep_attn = (uint32_t*)at(saved, L.off[S_KB]);
  return ENC_OK;
}

int enc_bwd_views(enc_ctx* ctx, const enc_dims* d, int dtype, void* scratch, enc_bwd_view* v) {
  if (!ctx) return ENC_ENULL;
  int r = check_dims(d, dtype);
  if (r) return r;
  if (!scratch || !v) return ENC_ENULL;
  const Layout L = bwd_layout(d, dtype);
  v->dY2 = at(scratch, L.off[B_DY2]);
  v->dA1 = at(scratch, L.off[B_DA1]);
  v->dh = at(scratch, L.off[B_DH]);
  v->dX1 = at(scratch, L.off[B_DX1]);
  v->dYo = at(scratch, L.off[B_DYO]);
  v->dC = at(scratch, L.off[B_DC]);
  v->dA = at(scratch, L.off[B_DA]);
  v->dS = at(scratch, L.off[B_DS]);
  v->dQKV = at(scratch, L.off[B_DQKV]);
  if (qkv_direct(ctx, d, dtype)) {
    const size_t ies = (size_t)d->I * esize(dtype);
    v->dQ = at(scratch, L.off[B_DQKV]);
    v->dK = at(scratch, L.off[B_DQKV] + ies);
    v->dV = at(scratch, L.off[B_DQKV] + 2 * ies);
    v->dqkv_ld = 3LL * d->I;
  } else {
    v->dQ = at(scratch, L.off[B_DQ]);
    v->dK = at(scratch, L.off[B_DK]);
    v->dV = at(scratch, L.off[B_DV]);
    v->dqkv_ld = d->P;
  }
  return ENC_OK;
}

// ------------------------------------------------------------------ per-operator ABI
int enc_dropout_mask(int64_t n, int64_t index0, float p, uint64_t seed, uint64_t subseq,
                     uint8_t* keep, enc_stream_t stream) {
  if (n < 0 || index0 < 0 || !valid_p(p)) return ENC_EINVAL;
  if (n > 0 && !keep) return ENC_ENULL;
  CK(launch_dropout_mask(n, index0, make_philox_key(p, seed, subseq), keep, (cudaStream_t)stream));
  return ENC_OK;
}

static int check_bjhp(int dtype, int B, int J, int H, int P) {
  if (!valid_dtype(dtype)) return ENC_EDTYPE;
  if (B < 0 || J <= 0 || H <= 0 || P <= 0) return ENC_EINVAL;
  if (P % 8) return ENC_EALIGN;
  if ((int64_t)B * J * 3 * H * P / 8 >= INT32_MAX) return ENC_EUNSUPPORTED;
  return ENC_OK;
}

int enc_aib_fwd(enc_ctx* ctx, int dtype, int B, int J, int H, int P, const void* qkv,
                const float* bqkv, void* q, void* k, void* v, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_bjhp(dtype, B, J, H, P);
  if (r) return r;
  CHECK_PTRS(qkv, bqkv, q, k, v);
  {
    OpTimer _t(ctx, ENC_OP_AIB_FWD, (cudaStream_t)stream, 1);
    CK(launch_aib_fwd(dtype, B, J, H, P, qkv, bqkv, q, k, v, (cudaStream_t)stream));
  }
  return ENC_OK;
}

int enc_aib_bwd(enc_ctx* ctx, int dtype, int B, int J, int H, int P, const void* dq,
                const void* dk, const void* dv, void* dqkv, float* dbqkv, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_bjhp(dtype, B, J, H, P);
  if (r) return r;
  CHECK_PTRS(dq, dk, dv, dqkv, dbqkv);
  {
    OpTimer _t(ctx, ENC_OP_AIB_BWD, (cudaStream_t)stream, 2);
    CK(launch_aib_bwd(dtype, B, J, H, P, dq, dk, dv, dqkv, dbqkv, ws_of(ctx), (cudaStream_t)stream));
  }
  return ENC_OK;
}

static int check_bhjk(int dtype, int B, int H, int J, int K, float p) {
  if (!valid_dtype(dtype)) return ENC_EDTYPE;
  if (B < 0 || H <= 0 || J <= 0 || K <= 0 || !valid_p(p)) return ENC_EINVAL;
  if (K % 8) return ENC_EALIGN;
  if (!rowop_supported(K)) return ENC_EUNSUPPORTED;
  if ((int64_t)B * H * J >= INT32_MAX) return ENC_EUNSUPPORTED;
  return ENC_OK;
}

int enc_bsb_fwd(enc_ctx* ctx, int dtype, int B, int H, int J, int K, float scale, const void* S,
                const float* mask_bias, float p, uint64_t seed, uint64_t subseq,
                int64_t batch_offset, void* P, void* A, int causal, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_bhjk(dtype, B, H, J, K, p);
  if (r) return r;
  if (batch_offset < 0 || (causal && J != K)) return ENC_EINVAL;
  CHECK_PTRS(S, P, A);
  if (mask_bias && !aligned16(mask_bias)) return ENC_EALIGN;
  {
    OpTimer _t(ctx, ENC_OP_BSB_FWD, (cudaStream_t)stream, 1);
    CK(launch_bsb_fwd(dtype, B, H, J, K, scale, S, mask_bias, make_philox_key(p, seed, subseq),
                      batch_offset, P, A, (cudaStream_t)stream, causal ? 1 : 0));
  }
  return ENC_OK;
}

int enc_bsb_bwd(enc_ctx* ctx, int dtype, int B, int H, int J, int K, float scale, const void* dA,
                const void* P, float p, uint64_t seed, uint64_t subseq, int64_t batch_offset,
                void* dS, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_bhjk(dtype, B, H, J, K, p);
  if (r) return r;
  if (batch_offset < 0) return ENC_EINVAL;
  CHECK_PTRS(dA, P, dS);
  {
    OpTimer _t(ctx, ENC_OP_BSB_BWD, (cudaStream_t)stream, 1);
    CK(launch_bsb_bwd(dtype, B, H, J, K, scale, dA, P, make_philox_key(p, seed, subseq),
                      batch_offset, dS, (cudaStream_t)stream));
  }
  return ENC_OK;
}

static int check_bjn(int dtype, int B, int J, int N, float p, bool rowop) {
  if (!valid_dtype(dtype)) return ENC_EDTYPE;
  if (B < 0 || J <= 0 || N <= 0 || !valid_p(p)) return ENC_EINVAL;
  if (N % 8) return ENC_EALIGN;
  if (rowop && !rowop_supported(N)) return ENC_EUNSUPPORTED;
  if ((int64_t)B * J * N / 8 >= INT32_MAX) return ENC_EUNSUPPORTED;
  return ENC_OK;
}

int enc_bdrln_fwd(enc_ctx* ctx, int dtype, int B, int J, int I, const void* Y, const float* bias,
                  const void* R, const float* gamma, const float* beta, float eps, float p,
                  uint64_t seed, uint64_t subseq, int64_t batch_offset, void* out, void* xhat,
                  float* rstd, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_bjn(dtype, B, J, I, p, true);
  if (r) return r;
  if (batch_offset < 0 || !(eps >= 0.f)) return ENC_EINVAL;
  CHECK_PTRS(Y, bias, R, gamma, beta, out, xhat, rstd);
  {
    OpTimer _t(ctx, ENC_OP_BDRLN_FWD1, (cudaStream_t)stream, 1);
    CK(launch_bdrln_fwd(dtype, B, J, I, Y, bias, R, gamma, beta, eps,
                        make_philox_key(p, seed, subseq), batch_offset, out, xhat, rstd,
                        (cudaStream_t)stream));
  }
  return ENC_OK;
}

int enc_bdrln_bwd(enc_ctx* ctx, int dtype, int B, int J, int I, const void* dOut,
                  const void* xhat, const float* rstd, const float* gamma, float p,
                  uint64_t seed, uint64_t subseq, int64_t batch_offset, void* dz, void* dYpre,
                  float* dgamma, float* dbeta, float* dbias, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_bjn(dtype, B, J, I, p, true);
  if (r) return r;
  if (!bdrln_bwd_supported(I, dtype)) return ENC_EUNSUPPORTED;
  if (batch_offset < 0) return ENC_EINVAL;
  CHECK_PTRS(dOut, xhat, rstd, gamma, dz, dYpre, dgamma, dbeta, dbias);
  {
    OpTimer _t(ctx, ENC_OP_BDRLN_BWD1, (cudaStream_t)stream, 2);
    CK(launch_bdrln_bwd(dtype, B, J, I, dOut, xhat, rstd, gamma, make_philox_key(p, seed, subseq),
                        batch_offset, dz, dYpre, dgamma, dbeta, dbias, ws_of(ctx),
                        (cudaStream_t)stream));
  }
  return ENC_OK;
}

int enc_bad_fwd(enc_ctx* ctx, int dtype, int B, int J, int U, const void* Y1, const float* b1,
                int act, float p, uint64_t seed, uint64_t subseq, int64_t batch_offset, void* h,
                void* A1, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_bjn(dtype, B, J, U, p, false);
  if (r) return r;
  if (batch_offset < 0 || act < 0 || act > 2) return ENC_EINVAL;
  CHECK_PTRS(Y1, b1, h, A1);
  {
    OpTimer _t(ctx, ENC_OP_BAD_FWD, (cudaStream_t)stream, 1);
    CK(launch_bad_fwd(dtype, B, J, U, Y1, b1, act, make_philox_key(p, seed, subseq), batch_offset,
                      h, A1, (cudaStream_t)stream));
  }
  return ENC_OK;
}

int enc_bad_bwd(enc_ctx* ctx, int dtype, int B, int J, int U, const void* dA1, const void* h,
                int act, float p, uint64_t seed, uint64_t subseq, int64_t batch_offset, void* dh,
                float* db1, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_bjn(dtype, B, J, U, p, false);
  if (r) return r;
  if (batch_offset < 0 || act < 0 || act > 2) return ENC_EINVAL;
  CHECK_PTRS(dA1, h, dh, db1);
  {
    OpTimer _t(ctx, ENC_OP_BAD_BWD, (cudaStream_t)stream, 2);
    CK(launch_bad_bwd(dtype, B, J, U, dA1, h, nullptr, act, make_philox_key(p, seed, subseq),
                      batch_offset, dh, db1, ws_of(ctx), (cudaStream_t)stream));
  }
  return ENC_OK;
}

int enc_attn_gemm(enc_ctx* ctx, int which, int B, int H, int J, int P, const void* X,
                  const void* Y, void* Z, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  if (which < ENC_AG_QK || which > ENC_AG_DK || B < 0 || H <= 0 || J <= 0 || P <= 0)
    return ENC_EINVAL;
  if (!attn_gemm_supported(J, P)) return ENC_EUNSUPPORTED;
  CHECK_PTRS(X, Y, Z);
  if (B == 0) return ENC_OK;
  // documented layouts: Q, K, V, dQ, dK, dV head-major (ld = P), C / dC token-major
  // [B,J,H,P] (ld = H*P)
  const int64_t hp = (int64_t)H * P;
  const int64_t ldx = which == ENC_AG_DA ? hp : P;
  const int64_t ldy = which == ENC_AG_DV ? hp : P;
  const int64_t ldz = which == ENC_AG_AV ? hp : P;
  CK(attn_contract(ctx, which, B, H, J, P, X, ldx, Y, ldy, Z, ldz, (cudaStream_t)stream));
  ctx->launches += 1;
  return ENC_OK;
}

int enc_attn_fwd_fused(enc_ctx* ctx, int B, int H, int J, int P, float scale, const void* Q,
                       const void* Kt, const float* mask_bias, float p, uint64_t seed,
                       uint64_t subseq, int64_t batch_offset, void* Pout, void* A,
                       uint32_t* keep_bits, int causal, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  if (B < 0 || H <= 0 || !valid_p(p) || batch_offset < 0) return ENC_EINVAL;
  if (!attn_fused_supported(J, P)) return ENC_EUNSUPPORTED;
  CHECK_PTRS(Q, Kt, Pout);   // A optional
  if (mask_bias && !aligned16(mask_bias)) return ENC_EALIGN;
  if (keep_bits && ((uintptr_t)keep_bits & 7u)) return ENC_EALIGN;
  if (B == 0) return ENC_OK;
  OpTimer _t(ctx, ENC_OP_BSB_FWD, (cudaStream_t)stream, 1);
  CK(launch_attn_qk_bsb(B, H, J, P, scale, Q, P, Kt, P, mask_bias,
                        make_philox_key(p, seed, subseq), batch_offset, Pout, A, keep_bits,
                        (cudaStream_t)stream, causal ? 1 : 0));
  return ENC_OK;
}

int enc_attn_keep_bits(enc_ctx* ctx, int B, int H, int J, int K, float p, uint64_t seed,
                       uint64_t subseq, int64_t batch_offset, uint32_t* keep_bits,
                       enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  if (B < 0 || H <= 0 || J <= 0 || K <= 0 || !valid_p(p) || batch_offset < 0) return ENC_EINVAL;
  if (K % 64) return ENC_EALIGN;
  if (!keep_bits) return ENC_ENULL;
  if ((uintptr_t)keep_bits & 7u) return ENC_EALIGN;
  if (B == 0) return ENC_OK;
  CK(launch_attn_keep_bits(B, H, J, K, make_philox_key(p, seed, subseq), batch_offset,
                           keep_bits, (cudaStream_t)stream));
  ctx->launches += 1;
  return ENC_OK;
}

int enc_attn_fwd_fused_bits(enc_ctx* ctx, int B, int H, int J, int P, float scale, const void* Q,
                            const void* Kt, const float* mask_bias, float p, uint64_t seed,
                            uint64_t subseq, int64_t batch_offset, void* Pout, void* A,
                            const uint32_t* keep_bits, int causal, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  if (B < 0 || H <= 0 || !valid_p(p) || batch_offset < 0) return ENC_EINVAL;
  if (!attn_fused_supported(J, P)) return ENC_EUNSUPPORTED;
  CHECK_PTRS(Q, Kt, Pout);
  if (!keep_bits) return ENC_ENULL;
  if (mask_bias && !aligned16(mask_bias)) return ENC_EALIGN;
  if ((uintptr_t)keep_bits & 7u) return ENC_EALIGN;
  if (B == 0) return ENC_OK;
  OpTimer _t(ctx, ENC_OP_BSB_FWD, (cudaStream_t)stream, 1);
  CK(launch_attn_qk_bsb(B, H, J, P, scale, Q, P, Kt, P, mask_bias,
                        make_philox_key(p, seed, subseq), batch_offset, Pout, A,
                        const_cast<uint32_t*>(keep_bits), (cudaStream_t)stream, causal ? 1 : 0,
                        1));
  return ENC_OK;
}

int enc_attn_bwd_fused(enc_ctx* ctx, int B, int H, int J, int P, float scale, const void* dC,
                       const void* V, const void* Pin, float p, uint64_t seed, uint64_t subseq,
                       int64_t batch_offset, const uint32_t* keep_bits, void* dS,
                       enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  if (B < 0 || H <= 0 || !valid_p(p) || batch_offset < 0) return ENC_EINVAL;
  if (!attn_fused_supported(J, P)) return ENC_EUNSUPPORTED;
  CHECK_PTRS(dC, V, Pin, dS);
  if (B == 0) return ENC_OK;
  OpTimer _t(ctx, ENC_OP_BSB_BWD, (cudaStream_t)stream, 1);
  CK(launch_attn_da_bsbb(B, H, J, P, scale, dC, (int64_t)H * P, V, P, Pin,
                         make_philox_key(p, seed, subseq), batch_offset, keep_bits, dS,
                         (cudaStream_t)stream));
  return ENC_OK;
}

int enc_attn_fwd_fused_av(enc_ctx* ctx, int B, int H, int J, int P, float scale, const void* Q,
                          const void* Kt, const void* V, const float* mask_bias, float p,
                          uint64_t seed, uint64_t subseq, int64_t batch_offset, void* Pout,
                          uint32_t* keep_bits, void* C, void* C_lo, int causal,
                          enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  if (B < 0 || H <= 0 || !valid_p(p) || batch_offset < 0) return ENC_EINVAL;
  if (!attn_fused_av_supported(J, P)) return ENC_EUNSUPPORTED;
  CHECK_PTRS(Q, Kt, V, Pout, C, C_lo);
  if (!keep_bits) return ENC_ENULL;
  if (mask_bias && !aligned16(mask_bias)) return ENC_EALIGN;
  if ((uintptr_t)keep_bits & 7u) return ENC_EALIGN;
  if (B == 0) return ENC_OK;
  OpTimer _t(ctx, ENC_OP_BSB_FWD, (cudaStream_t)stream, 1);
  CK(launch_attn_qk_bsb_av(B, H, J, P, scale, Q, P, Kt, P, V, P, mask_bias,
                           make_philox_key(p, seed, subseq), batch_offset, Pout, keep_bits, C,
                           C_lo, (int64_t)H * P, (cudaStream_t)stream, causal ? 1 : 0));
  return ENC_OK;
}

int enc_attn_bwd_fused_dc(enc_ctx* ctx, int B, int H, int J, int P, float scale, const void* dC,
                          const void* V, const void* Pin, const void* C_hi, const void* C_lo,
                          float p, uint64_t seed, uint64_t subseq, int64_t batch_offset,
                          const uint32_t* keep_bits, void* dS, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  if (B < 0 || H <= 0 || !valid_p(p) || batch_offset < 0) return ENC_EINVAL;
  if (!attn_fused_supported(J, P)) return ENC_EUNSUPPORTED;
  CHECK_PTRS(dC, V, Pin, C_hi, C_lo, dS);
  if (B == 0) return ENC_OK;
  OpTimer _t(ctx, ENC_OP_BSB_BWD, (cudaStream_t)stream, 1);
  CK(launch_attn_da_bsbb(B, H, J, P, scale, dC, (int64_t)H * P, V, P, Pin,
                         make_philox_key(p, seed, subseq), batch_offset, keep_bits, dS,
                         (cudaStream_t)stream, false, C_hi, C_lo, (int64_t)H * P));
  return ENC_OK;
}

int enc_set_option(enc_ctx* ctx, int key, int value) {
  if (!ctx) return ENC_ENULL;
  if (key == ENC_OPT_ATTN_TC) {
    ctx->attn_tc = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_GEMM_LT) {
    ctx->use_lt = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_GEMM_AUTOTUNE) {
    if (ctx->lt) lt_set_autotune(ctx->lt, value ? 1 : 0);
    return ENC_OK;
  }
  if (key == ENC_OPT_ATTN_FUSED) {
    ctx->attn_fused = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_ATTN_BH) {
    ctx->attn_bh = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_QKV_DIRECT) {
    ctx->qkv_direct = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_BWD_SIDE) {
    if (value < 0 || value > 3) return ENC_EINVAL;
    // 1: weight-gradient contractions on the side stream; 2: and the attention half's
    // column-sum finalize on a second one; 3: only the finalize on the second stream
    ctx->bwd_side = value;
    return ENC_OK;
  }
  if (key == ENC_OPT_ATTN_OVERLAP) {
    ctx->attn_overlap = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_GEMM_TC) {
    ctx->gemm_tc = value ? 0xFFFFFFFFu : 0u;
    return ENC_OK;
  }
  if (key == ENC_OPT_GEMM_TC_MASK) {
    ctx->gemm_tc = (uint32_t)value;
    return ENC_OK;
  }
  if (key == ENC_OPT_QKV_FUSION) {
    if (value < ENC_QKV_SEPARATE || value > ENC_QKV_KV_STACKED) return ENC_EINVAL;
    ctx->qkv_fusion = value;
    ctx->qkv_fusion_bwd = value;
    return ENC_OK;
  }
  if (key == ENC_OPT_QKV_FUSION_BWD) {
    if (value < ENC_QKV_SEPARATE || value > ENC_QKV_KV_STACKED) return ENC_EINVAL;
    ctx->qkv_fusion_bwd = value;
    return ENC_OK;
  }
  if (key == ENC_OPT_BDRLN_VARIANT) {
    for (int site = 0; site < 4; ++site)
      if (((value >> (4 * site)) & 15) > 5) return ENC_EINVAL;
    if (value < 0 || value >= (1 << 16)) return ENC_EINVAL;
    ctx->bdrln_variant = value;
    return ENC_OK;
  }
  if (key == ENC_OPT_KEEP_AHEAD) {
    ctx->keep_ahead = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_ATTN_DC) {
    ctx->attn_dc = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_MASK_BYTES) {
    ctx->mask_bytes = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_ATTN_FUSED_AV) {
    ctx->attn_fused_av = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_SIDE_OPS) {
    ctx->side_ops = (uint32_t)value;
    return ENC_OK;
  }
  if (key == ENC_OPT_MASK_AHEAD) {
    if (value < 0 || value > 2) return ENC_EINVAL;
    ctx->mask_ahead = value;   // 2: the BDRLN sites' bytes too
    return ENC_OK;
  }
  if (key == ENC_OPT_AV_KEEP_GEN) {
    ctx->av_keep_gen = value ? 1 : 0;
    return ENC_OK;
  }
  if (key == ENC_OPT_PDL) {
    if (value < 0 || value > 31) return ENC_EINVAL;
    pdl_set(value);
    return ENC_OK;
  }
  if (key == ENC_OPT_GEMM_PAIR) {
    ctx->gemm_cg = value ? 0 : 1;
    return ENC_OK;
  }
  return ENC_EINVAL;
}

int enc_wgemm(enc_ctx* ctx, int M, int N, int K, const void* A, int64_t lda, int tA,
              const void* B, int64_t ldb, int tB, void* C, int64_t ldc, int c_dtype, int beta,
              const float* bias, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  if (!valid_dtype(c_dtype)) return ENC_EDTYPE;
  if (M <= 0 || N <= 0 || K <= 0 || (beta != 0 && beta != 1) || (beta && c_dtype == ENC_FP32))
    return ENC_EINVAL;
  if (lda < (tA ? M : K) || ldb < (tB ? K : N) || ldc < N) return ENC_EINVAL;
  if (N % 8 || K % 8 || lda % 8 || ldb % 8 || ldc % (c_dtype == ENC_FP32 ? 4 : 8))
    return ENC_EALIGN;
  if (lda > INT32_MAX || ldb > INT32_MAX || ldc > INT32_MAX) return ENC_EUNSUPPORTED;
  CHECK_PTRS(A, B, C);
  if (bias && !aligned16(bias)) return ENC_EALIGN;
  WgemmArgs g;
  g.M = M; g.N = N; g.K = K;
  g.A = A; g.lda = lda; g.a_mn = tA ? 1 : 0;
  g.B = B; g.ldb = ldb; g.b_mn = tB ? 0 : 1;
  g.C = C; g.ldc = ldc; g.out_f32 = c_dtype == ENC_FP32;
  g.beta = beta;
  g.bias = bias;
  g.ws = ctx->wg_ws;
  g.ws_bytes = ctx->wg_ws_bytes;
  g.cg = ctx->gemm_cg;
  if (!wgemm_supported(g)) return ENC_EUNSUPPORTED;
  CK(launch_wgemm(g, ctx->num_sms, (cudaStream_t)stream));
  ctx->launches += wgemm_launches(g, ctx->num_sms);
  return ENC_OK;
}

static int check_ffn_call(int B, int J, int I, int U, float p, int act, int64_t boff) {
  if (B <= 0 || J <= 0 || I <= 0 || U <= 0 || !valid_p(p) || act < 0 || act > 2 || boff < 0)
    return ENC_EINVAL;
  if (I % 8 || U % 8) return ENC_EALIGN;
  if ((int64_t)B * J * U / 8 >= INT32_MAX) return ENC_EUNSUPPORTED;
  return ENC_OK;
}

int enc_linear1_bad_fwd(enc_ctx* ctx, int B, int J, int I, int U, const void* X1,
                        const void* W1, const float* b1, int act, float p, uint64_t seed,
                        uint64_t subseq, int64_t batch_offset, void* h, void* A1,
                        enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_ffn_call(B, J, I, U, p, act, batch_offset);
  if (r) return r;
  CHECK_PTRS(X1, W1, b1, h, A1);
  enc_dims d{B, J, J, 1, I, I, I, U};
  enc_cfg cfg{};
  cfg.act = act;
  cfg.batch_offset = batch_offset;
  // the fused kernel regardless of ENC_OPT_GEMM_TC
  WgemmArgs g = ffn_fwd_args(ctx, &d, ENC_BF16, &cfg, X1, W1, b1,
                             make_philox_key(p, seed, subseq), h, A1, true);
  if (!wgemm_supported(g)) return ENC_EUNSUPPORTED;
  OpTimer _t(ctx, ENC_OP_GEMM_L1, (cudaStream_t)stream, 1);
  CK(launch_wgemm(g, ctx->num_sms, (cudaStream_t)stream));
  return ENC_OK;
}

int enc_linear2_dx_bad_bwd(enc_ctx* ctx, int B, int J, int I, int U, const void* dY2,
                           const void* W2, const void* h, int act, float p, uint64_t seed,
                           uint64_t subseq, int64_t batch_offset, void* dh, float* db1,
                           enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_ffn_call(B, J, I, U, p, act, batch_offset);
  if (r) return r;
  CHECK_PTRS(dY2, W2, h, dh, db1);
  enc_dims d{B, J, J, 1, I, I, I, U};
  enc_cfg cfg{};
  cfg.act = act;
  cfg.batch_offset = batch_offset;
  WgemmArgs g = ffn_bwd_args(ctx, &d, ENC_BF16, &cfg, dY2, W2, h,
                             make_philox_key(p, seed, subseq), dh, ctx->red, true);
  const int R = wgemm_partial_rows(g);
  if ((size_t)R * U > ctx->red_floats) return ENC_EUNSUPPORTED;
  if (!wgemm_supported(g)) return ENC_EUNSUPPORTED;
  OpTimer _t(ctx, ENC_OP_GEMM_L2_DX, (cudaStream_t)stream, 2);
  CK(launch_wgemm(g, ctx->num_sms, (cudaStream_t)stream));
  CK(launch_colsum_finalize(ctx->red, R, U, U, db1, nullptr, nullptr, (cudaStream_t)stream));
  return ENC_OK;
}

int enc_bei(enc_ctx* ctx, int dtype, int64_t n, const void* a, const void* b, void* out,
            enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  if (!valid_dtype(dtype)) return ENC_EDTYPE;
  if (n < 0) return ENC_EINVAL;
  if (n % 8) return ENC_EALIGN;
  CHECK_PTRS(a, b, out);
  CK(launch_bei(dtype, n, a, b, out, (cudaStream_t)stream));
  return ENC_OK;
}

// ------------------------------------------------------------------ whole layer
static int check_params(const enc_params* p) {
  if (!p) return ENC_ENULL;
  CHECK_PTRS(p->Wqkv, p->Wo, p->W1, p->W2, p->bqkv, p->bo, p->b1, p->b2, p->g1, p->be1, p->g2,
             p->be2);
  return ENC_OK;
}

int encoder_layer_forward(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                          const enc_params* prm, const void* X, const float* mask_bias, void* Y,
                          void* saved, void* scratch, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_dims(d, dtype);
  if (r) return r;
  if ((r = check_cfg(cfg))) return r;
  if ((r = check_params(prm))) return r;
  CHECK_PTRS(X, Y, saved, scratch);
  if (mask_bias && !aligned16(mask_bias)) return ENC_EALIGN;
  if (d->B == 0) return ENC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CB(cublasSetStream(ctx->blas, st));
  const int B = d->B, J = d->J, K = d->K, H = d->H, P = d->P, I = d->I, U = d->U;
  const int BJ = B * J, BH = B * H;
  const size_t es = esize(dtype);
  const Layout SL = saved_layout(d, dtype), FL = fwd_layout(d, dtype);
  void *Q = at(saved, SL.off[S_Q]), *Kt = at(saved, SL.off[S_K]), *V = at(saved, SL.off[S_V]);
  void *Pm = at(saved, SL.off[S_P]), *A = at(saved, SL.off[S_A]), *C = at(saved, SL.off[S_C]);
  void *X1 = at(saved, SL.off[S_X1]), *xh1 = at(saved, SL.off[S_XH1]);
  void *h = at(saved, SL.off[S_H]), *A1 = at(saved, SL.off[S_A1]);
  void* xh2 = at(saved, SL.off[S_XH2]);
  float *r1 = (float*)at(saved, SL.off[S_R1]), *r2 = (float*)at(saved, SL.off[S_R2]);
  void** ptr = (void**)at(scratch, FL.off[F_PTR]);
  void *QKV = at(scratch, FL.off[F_QKV]), *S = at(scratch, FL.off[F_S]);
  void* Yo = at(scratch, FL.off[F_YO]);
  void* Y2 = at(scratch, FL.off[F_Y2]);
  const uint64_t l4 = 4ull * cfg->layer_id;
  const float scale = 1.0f / sqrtf((float)P);  // DESIGN.md R3
  const int64_t boff = cfg->batch_offset;
  const bool tc_attn = tc_attn_of(ctx, dtype, J, P);
  const bool fused_attn = tc_attn && ctx->attn_fused && attn_fused_supported(J, P);
  // tcgen05 paths: Q, K, V are read in place from the QKV contraction output (row stride
  // 3I, spanning the saved Q, K, V regions); the AIB bias rides in the contraction epilogue
  const bool direct = qkv_direct(ctx, d, dtype);
  const int64_t ldqkv = direct ? 3LL * I : P;
  void* QKVs = Q;
  if (direct) {
    Kt = (char*)QKVs + (size_t)I * es;
    V = (char*)QKVs + 2 * (size_t)I * es;
    if (SL.off[S_K] != SL.off[S_Q] + (size_t)BJ * I * es ||
        SL.off[S_V] != SL.off[S_K] + (size_t)BJ * I * es)
      return ENC_EUNSUPPORTED;   // Q, K, V regions not contiguous (cannot happen: J % 128 == 0)
  }

  // fused path: the attention keep words (4.2 MB at config L) are generated on the side
  // stream while the QKV contraction runs (it leaves the FMA pipe idle), so the fused score
  // kernel reads them instead of running Philox between its MMA and its epilogue
  const PhiloxKey pk_attn = make_philox_key(cfg->p_attn, cfg->seed, l4 + 0);
  uint32_t* kbits = (uint32_t*)at(saved, SL.off[S_KB]);
  const bool keep_ahead = fused_attn && ctx->keep_ahead && ctx->side && K % 64 == 0;
  if (keep_ahead) {
    CK(cudaEventRecord(ctx->ev_kb_fork, st));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_kb_fork, 0));
    CK(launch_attn_keep_bits(B, H, J, K, pk_attn, boff, kbits, ctx->side));
    ctx->launches += 1;
    CK(cudaEventRecord(ctx->ev_kb_join, ctx->side));
  }
  // Q,K,V (Table A.1 :549): QKV[BJ,3I] = X Wqkv^T (+ bqkv, AIB :550, on the direct path),
  // as one contraction per group of stacked weight blocks (algebraic fusion, Table A.2,
  // Q, K, V separate / QK stacked + V / QKV stacked (default) / Q + KV
  // stacked), each writing its column blocks of QKV (row stride 3I).  cuBLASLt takes a bf16
  // output's bias in bf16: rounded to bf16 for its epilogue (R18; one cast kernel).
  int ngrp = 0, gstart[3], gcount[3];
  qkv_groups(ctx->qkv_fusion, &ngrp, gstart, gcount);
  bool bias_done = false;
  {
    OpTimer _t(ctx, ENC_OP_GEMM_QKV, st, 0);
    void* qkv_out = direct ? QKVs : QKV;
    bool cast_done = false;
    for (int gi = 0; gi < ngrp; ++gi) {
      const int s0 = gstart[gi], nI = gcount[gi] * I;
      const void* Wg = (const char*)prm->Wqkv + (size_t)s0 * I * I * es;
      void* Cg = (char*)qkv_out + (size_t)s0 * I * es;
      bool done = false;
      if (direct && (gi == 0 || bias_done)) {   // tcgen05: the fp32 bias in its epilogue
        r = wcontract(ctx, ENC_OP_GEMM_QKV, st, dtype, dtype, false, true, BJ, nI, I, X, I, Wg,
                      I, 0.f, Cg, 3 * I, prm->bqkv + (size_t)s0 * I);
        if (r == ENC_OK) done = true;
        else if (r != ENC_EUNSUPPORTED) return r;
      }
      if (!done && direct && (gi == 0 || bias_done) && ctx->lt && ctx->use_lt &&
          ctx->red_floats >= (size_t)3 * I) {
        if (!cast_done) {
          CK(launch_f32_to_bf16(3 * I, prm->bqkv, ctx->red, st));
          ctx->launches += 1;
          cast_done = true;
        }
        done = wgemm_epi(ctx, st, dtype, dtype, false, true, BJ, nI, I, X, I, Wg, I, Cg, 3 * I,
                         LT_EPI_BIAS, (float*)((char*)ctx->red + (size_t)s0 * I * 2));
      }
      if (gi == 0) bias_done = done;
      if (done != bias_done) return ENC_EUNSUPPORTED;   // every group the same way
      if (!done)
        if ((r = wcontract(ctx, ENC_OP_GEMM_QKV, st, dtype, dtype, false, true, BJ, nI, I, X, I,
                           Wg, I, 0.f, Cg, 3 * I)))
          return r;
    }
  }
  // AIB (:550): in place on the direct path unless the epilogue added the bias
  {
    OpTimer _t(ctx, ENC_OP_AIB_FWD, st, direct && bias_done ? 0 : 1, !(direct && bias_done));
    if (!direct)
      CK(launch_aib_fwd(dtype, B, J, H, P, QKV, prm->bqkv, Q, Kt, V, st));
    else if (!bias_done)
      CK(launch_bias_rows(dtype, BJ, 3 * I, QKVs, prm->bqkv, st));
  }
  // R29: the FFN site's keep bytes are drawn by a small kernel on the side stream, made
  // ready together with the fused score kernel (launched at high priority): its CTAs take the
  // SMs the score kernel's last wave leaves idle; Linear1 + BAD then reads the bytes
  const PhiloxKey pk_ffn = make_philox_key(cfg->p_ffn, cfg->seed, l4 + 2);
  // (without the fused score + A.V kernel's spare SMs the side kernel measured slower: R29)
  const int spare_sms = ctx->num_sms - balanced_grid((J / 128) * B * H);
  const bool mask_ahead = ctx->mask_ahead && fused_attn && ctx->side &&
                          bad_bytes_of(ctx, d, dtype) && ((size_t)BJ * (U / 8)) % 4 == 0 &&
                          ctx->attn_fused_av && attn_fused_av_supported(J, P) && spare_sms > 0 &&
                          dc_term_of(ctx, fused_attn, J, P) && use_bh(ctx, J, P) &&
                          !ctx->keep_ahead && !ctx->av_keep_gen;
  // R31: beside the fused score + A.V kernel, launched on a balanced grid (512 tiles: 128
  // CTAs x 4), the keep bytes of the FFN site and of both BDRLN sites are drawn by 1024-thread
  // CTAs on the SMs it leaves free (its CTAs hold every register of theirs, so the two never
  // share an SM)
  const bool spare_ahead = mask_ahead && ((size_t)BJ * (I / 8)) % 4 == 0;
  const bool ln_ahead = spare_ahead && ctx->mask_ahead == 2;   // BDRLN sites too
  if (mask_ahead) {
    CK(cudaEventRecord(ctx->ev_mk_fork, st));
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_mk_fork, 0));
    const int cap = spare_ahead ? spare_sms : 0;
    CK(launch_keep_bytes((int64_t)BJ * (U / 8), boff * (int64_t)J * (U / 8), pk_ffn,
                         (uint8_t*)at(saved, SL.off[S_KBF]), ctx->side, cap));
    ctx->launches += 1;
    if (spare_ahead && ctx->mask_ahead == 2) {   // (measured: does not fit the window)
      for (int site = 0; site < 2; ++site) {
        CK(launch_keep_bytes((int64_t)BJ * (I / 8), boff * (int64_t)J * (I / 8),
                             make_philox_key(cfg->p_hidden, cfg->seed, l4 + 1 + 2 * site),
                             (uint8_t*)at(saved, SL.off[site ? S_KB2 : S_KB1]), ctx->side,
                             cap));
        ctx->launches += 1;
      }
    }
    CK(cudaEventRecord(ctx->ev_mk_join, ctx->side));
  }
  // fused + per-(b, h) path: A = dropout(P) is never stored -- the A V (and backward
  // A^T dC) contraction applies the stored keep bits to P while it is in shared memory
  const bool drop_on_load = fused_attn && use_bh(ctx, J, P);
  // R28: on that path the A.V kernel's dropout-on-load warps generate the keep words from
  // the Philox stream (FMA work beside a memory-bound stream) and store them for the
  // backward; the score kernel runs no Philox (ENC_OPT_AV_KEEP_GEN, not with keep-ahead)
  const bool av_gen = drop_on_load && ctx->av_keep_gen && !keep_ahead;
  // R30: QK^T + BSB + A.V in one kernel (P aliased as the A operand in TMEM); C's low word
  // is stored with C, so the backward's row term (R26) needs the same saved layout
  const bool fused_av = drop_on_load && ctx->attn_fused_av && !keep_ahead && !av_gen &&
                        attn_fused_av_supported(J, P) && dc_term_of(ctx, fused_attn, J, P);
  if (fused_av) {
    OpTimer _t(ctx, ENC_OP_BSB_FWD, st, 1);
    CK(launch_attn_qk_bsb_av(B, H, J, P, scale, Q, ldqkv, Kt, ldqkv, V, ldqkv, mask_bias,
                             pk_attn, boff, Pm, kbits, C, at(saved, SL.off[S_CLO]), I, st,
                             cfg->causal ? 1 : 0));
  } else if (fused_attn) {
    // QK^T (:551) + BSB (:552) in one tcgen05 kernel: S stays in TMEM
    if (keep_ahead) CK(cudaStreamWaitEvent(st, ctx->ev_kb_join, 0));
    OpTimer _t(ctx, ENC_OP_BSB_FWD, st, 1);
    // (A.V generates the keep words on load, R28: the score kernel then writes P only)
    CK(launch_attn_qk_bsb(B, H, J, P, scale, Q, ldqkv, Kt, ldqkv, mask_bias, pk_attn, boff, Pm,
                          drop_on_load ? nullptr : A, av_gen ? nullptr : kbits, st,
                          cfg->causal ? 1 : 0, keep_ahead ? 1 : 0, mask_ahead));
  } else {
    // QK^T (:551): S_bh[J,K] = Q_bh K_bh^T
    {
      OpTimer _t(ctx, ENC_OP_GEMM_QK, st, tc_attn ? 1 : 0);
      if (tc_attn)
        CK(launch_attn_gemm(ENC_AG_QK, B, H, J, P, Q, ldqkv, Kt, ldqkv, S, 0, st));
      else
        CB(gemm_rm_strided(ctx->blas, dtype, false, true, J, K, P, 1.f, Q, P, (long long)J * P,
                           Kt, P, (long long)K * P, 0.f, S, K, (long long)J * K, BH));
    }
    // BSB (:552)
    {
      OpTimer _t(ctx, ENC_OP_BSB_FWD, st, 1);
      CK(launch_bsb_fwd(dtype, B, H, J, K, scale, S, mask_bias,
                        make_philox_key(cfg->p_attn, cfg->seed, l4 + 0), boff, Pm, A, st,
                        cfg->causal ? 1 : 0));
    }
  }
  // Gamma (:553): C_bh[J,P] = A_bh V_bh, written into C[B,J,H,P]
  {
    OpTimer _t(ctx, ENC_OP_GEMM_AV, st, fused_av ? 0 : 1, !fused_av);
    if (fused_av) {
      // computed by the score kernel above (R30)
    } else if (drop_on_load) {
      // (+ the fp32 result's low bf16 word for the backward's row term, R26)
      CK(launch_attn_av_bh(B, H, J, P, Pm, V, ldqkv, C, I, kbits, pk_attn.scale, st,
                           dc_term_of(ctx, fused_attn, J, P) ? at(saved, SL.off[S_CLO])
                                                             : nullptr,
                           av_gen ? &pk_attn : nullptr, boff));
    } else if (tc_attn) {
      CK(attn_contract(ctx, ENC_AG_AV, B, H, J, P, A, 0, V, ldqkv, C, I, st));
    } else {
      CK(launch_make_attn_ptrs(B, H, J, P, es, A, V, C, nullptr, nullptr, ptr, st));
      CB(gemm_rm_batched(ctx->blas, dtype, false, false, J, P, K, 1.f, (const void* const*)ptr, K,
                         (const void* const*)(ptr + BH), P, 0.f, (void* const*)(ptr + 2 * BH), I,
                         BH));
    }
  }
  // Out (:554)
  {
    OpTimer _t(ctx, ENC_OP_GEMM_OUT, st, 0);
    if ((r = wcontract(ctx, ENC_OP_GEMM_OUT, st, dtype, dtype, false, true, BJ, I, I, C, I, prm->Wo, I, 0.f, Yo, I)))
      return r;
  }
  // BDRLN site 1 (:555-558)
  {
    OpTimer _t(ctx, ENC_OP_BDRLN_FWD1, st, 1);
    if (ln_ahead) CK(cudaStreamWaitEvent(st, ctx->ev_mk_join, 0));
    CK(launch_bdrln_fwd(dtype, B, J, I, Yo, prm->bo, X, prm->g1, prm->be1, cfg->ln_eps,
                        make_philox_key(cfg->p_hidden, cfg->seed, l4 + 1), boff, X1, xh1, r1, st,
                        ctx->bdrln_variant & 15,
                        ctx->mask_bytes && !ln_ahead ? (uint8_t*)at(saved, SL.off[S_KB1])
                                                     : nullptr,
                        ln_ahead ? (const uint8_t*)at(saved, SL.off[S_KB1]) : nullptr));
  }
  // Linear (:559) + BAD (:560-562).  The activation input h = X1 W1^T + b1 is kept for the
  // backward (saved.h); on the tcgen05 path BAD runs in the contraction's epilogue
  WgemmArgs l1 = ffn_fwd_args(ctx, d, dtype, cfg, X1, prm->W1, prm->b1, pk_ffn, h, A1);
  if (mask_ahead) {
    CK(cudaStreamWaitEvent(st, ctx->ev_mk_join, 0));
    l1.kb_in = (const uint8_t*)at(saved, SL.off[S_KBF]);
  } else if (bad_bytes_of(ctx, d, dtype)) {
    l1.kb_out = (uint8_t*)at(saved, SL.off[S_KBF]);
  }
  if (wgemm_supported(l1)) {
    // (BAD has no launch of its own: no ENC_OP_BAD_FWD timing on this path)
    OpTimer _t(ctx, ENC_OP_GEMM_L1, st, 1);
    CK(launch_wgemm(l1, ctx->num_sms, st));
  } else {
    {
      OpTimer _t(ctx, ENC_OP_GEMM_L1, st, 0);
      if ((r = wcontract(ctx, ENC_OP_GEMM_L1, st, dtype, dtype, false, true, BJ, U, I, X1, I, prm->W1, I, 0.f, h,
                         U)))
        return r;
    }
    OpTimer _t(ctx, ENC_OP_BAD_FWD, st, 1);   // h = Y1 + b1 in place, A1
    CK(launch_bad_fwd(dtype, B, J, U, h, prm->b1, cfg->act, pk_ffn, boff, h, A1, st));
  }
  // Linear (:563)
  {
    OpTimer _t(ctx, ENC_OP_GEMM_L2, st, 0);
    if ((r = wcontract(ctx, ENC_OP_GEMM_L2, st, dtype, dtype, false, true, BJ, I, U, A1, U, prm->W2, U, 0.f, Y2, I)))
      return r;
  }
  // BDRLN site 2 (:564-567)
  {
    OpTimer _t(ctx, ENC_OP_BDRLN_FWD2, st, 1);
    CK(launch_bdrln_fwd(dtype, B, J, I, Y2, prm->b2, X1, prm->g2, prm->be2, cfg->ln_eps,
                        make_philox_key(cfg->p_hidden, cfg->seed, l4 + 3), boff, Y, xh2, r2, st,
                        (ctx->bdrln_variant >> 4) & 15,
                        ctx->mask_bytes && !ln_ahead ? (uint8_t*)at(saved, SL.off[S_KB2])
                                                     : nullptr,
                        ln_ahead ? (const uint8_t*)at(saved, SL.off[S_KB2]) : nullptr));
  }
  {
    std::lock_guard<std::mutex> lk(ctx->mu);
    if (ctx->saved_paths.size() > 4096) ctx->saved_paths.clear();
    ctx->saved_paths[saved] = path_flags(ctx, d, dtype);
  }
  return ENC_OK;
}

// parts: bit 0 = FFN half (BDRLN-bwd#2 .. Linear1 dW: all FFN-parameter gradients final),
//        bit 1 = attention half (BDRLN-bwd#1 .. QKV dW)
static int backward_impl(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                         const enc_params* prm, const void* X, const void* saved,
                         const void* dY, void* dX, const enc_grads* g, void* scratch,
                         enc_stream_t stream, int parts) {
  if (!ctx) return ENC_ENULL;
  if (parts < 1 || parts > 3) return ENC_EINVAL;
  int r = check_dims(d, dtype);
  if (r) return r;
  if ((r = check_cfg(cfg))) return r;
  if ((r = check_params(prm))) return r;
  if (!g) return ENC_ENULL;
  CHECK_PTRS(X, saved, dY, dX, scratch, g->dWqkv, g->dWo, g->dW1, g->dW2, g->dbqkv, g->dbo, g->db1,
             g->db2, g->dg1, g->dbe1, g->dg2, g->dbe2);
  {
    // the saved set must be read with the attention path it was written with
    std::lock_guard<std::mutex> lk(ctx->mu);
    auto it = ctx->saved_paths.find(saved);
    if (it != ctx->saved_paths.end() && it->second != path_flags(ctx, d, dtype))
      return ENC_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int B = d->B, J = d->J, K = d->K, H = d->H, P = d->P, I = d->I, U = d->U;
  const int BJ = B * J, BH = B * H;
  const size_t es = esize(dtype);
  const ReduceWs ws = ws_of(ctx);
  if (B == 0) {
    const size_t n[12] = {(size_t)3 * I * I, (size_t)I * I, (size_t)U * I, (size_t)I * U,
                          (size_t)3 * I, (size_t)I, (size_t)U, (size_t)I, (size_t)I, (size_t)I,
                          (size_t)I, (size_t)I};
    float* p[12] = {g->dWqkv, g->dWo, g->dW1, g->dW2, g->dbqkv, g->dbo,
                    g->db1,   g->db2, g->dg1, g->dbe1, g->dg2, g->dbe2};
    for (int i = 0; i < 12; ++i) CK(cudaMemsetAsync(p[i], 0, n[i] * sizeof(float), st));
    return ENC_OK;
  }
  CB(cublasSetStream(ctx->blas, st));
  const Layout SL = saved_layout(d, dtype), BL = bwd_layout(d, dtype);
  void* sv = (void*)saved;
  void *Q = at(sv, SL.off[S_Q]), *Kt = at(sv, SL.off[S_K]), *V = at(sv, SL.off[S_V]);
  void *Pm = at(sv, SL.off[S_P]), *A = at(sv, SL.off[S_A]), *C = at(sv, SL.off[S_C]);
  void *X1 = at(sv, SL.off[S_X1]), *xh1 = at(sv, SL.off[S_XH1]);
  void *h = at(sv, SL.off[S_H]), *A1 = at(sv, SL.off[S_A1]), *xh2 = at(sv, SL.off[S_XH2]);
  float *r1 = (float*)at(sv, SL.off[S_R1]), *r2 = (float*)at(sv, SL.off[S_R2]);
  void** ptr = (void**)at(scratch, BL.off[B_PTR]);
  void *dY2 = at(scratch, BL.off[B_DY2]), *dA1 = at(scratch, BL.off[B_DA1]);
  void *dh = at(scratch, BL.off[B_DH]), *dX1 = at(scratch, BL.off[B_DX1]);
  void *dYo = at(scratch, BL.off[B_DYO]), *dC = at(scratch, BL.off[B_DC]);
  void *dA = at(scratch, BL.off[B_DA]), *dS = at(scratch, BL.off[B_DS]);
  void *dQ = at(scratch, BL.off[B_DQ]), *dK = at(scratch, BL.off[B_DK]);
  void *dV = at(scratch, BL.off[B_DV]), *dQKV = at(scratch, BL.off[B_DQKV]);
  const uint64_t l4 = 4ull * cfg->layer_id;
  const float scale = 1.0f / sqrtf((float)P);
  const int64_t boff = cfg->batch_offset;
  const bool tc_attn = tc_attn_of(ctx, dtype, J, P);
  const bool fused_attn = tc_attn && ctx->attn_fused && attn_fused_supported(J, P);
  const int F32 = ENC_FP32;
  // direct QKV layout (see forward): Q, K, V read from the QKV tensor, dQ, dK, dV written
  // straight into the column blocks of dQKV, row stride 3I
  const bool direct = qkv_direct(ctx, d, dtype);
  const int64_t ldqkv = direct ? 3LL * I : P;
  if (direct) {
    Kt = (char*)Q + (size_t)I * es;
    V = (char*)Q + 2 * (size_t)I * es;
    dQ = dQKV;
    dK = (char*)dQKV + (size_t)I * es;
    dV = (char*)dQKV + 2 * (size_t)I * es;
  }

  // The column sums of each half are finished by one batched finalize launch at the end of
  // the half (deferred jobs, disjoint partial regions of the reduction workspace).
  auto after = [&](const ColsumJob& j) {   // workspace past a recorded job's partials
    float* base = const_cast<float*>(j.partials) + (((size_t)j.R * j.ncols + 63) & ~(size_t)63);
    return ReduceWs{base, ws.cap_floats - (size_t)(base - ws.partials), ws.num_sms};
  };
  // whole backward in one call: the FFN half's column sums are finished in the attention
  // half's finalize launch (one launch per step; the split call finishes them early so the
  // FFN bucket can be all-reduced while the attention half runs)
  const bool ffn_deferred = (parts & 3) == 3;
  ColsumJob ffn_jobs[2];
  // weight-gradient contractions go to the side stream: fork once the inputs exist, join
  // before returning (the next forward reuses the scratch they read)
  const bool use_side = (ctx->bwd_side == 1 || ctx->bwd_side == 2) && ctx->lt && ctx->use_lt &&
                        ctx->side;
  bool forked = false;
  // ENC_OPT_SIDE_OPS: a mask of weight-gradient contractions put on the side stream
  // (overrides ENC_OPT_BWD_SIDE's all-or-none for those it names)
  auto fork_op = [&](int op) -> bool {
    return ctx->side && ctx->lt && ctx->use_lt && ((ctx->side_ops >> op) & 1u);
  };
  auto fork = [&](int op = -1) -> cudaStream_t {
    if (!use_side && !(op >= 0 && fork_op(op))) return st;
    cudaEventRecord(ctx->ev_fork, st);
    cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0);
    forked = true;
    return ctx->side;
  };
  auto join = [&]() -> cudaError_t {
    if (!forked) return cudaSuccess;
    forked = false;
    cudaError_t e = cudaEventRecord(ctx->ev_join, ctx->side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ctx->ev_join, 0);
    return e;
  };
  if (parts & 1) {
  // BDRLN-bwd site 2 (:570-572, bias2 dW :575): dz2 -> dX1 (residual path), dY2
  {
    OpTimer _t(ctx, ENC_OP_BDRLN_BWD2, st, 1);
    ReduceWs w = ws;
    w.defer = &ffn_jobs[0];
    CK(launch_bdrln_bwd(dtype, B, J, I, dY, xh2, r2, prm->g2,
                        make_philox_key(cfg->p_hidden, cfg->seed, l4 + 3), boff, dX1, dY2, g->dg2,
                        g->dbe2, g->db2, w, st, (ctx->bdrln_variant >> 8) & 15,
                        ctx->mask_bytes ? (const uint8_t*)at(sv, SL.off[S_KB2]) : nullptr));
  }
  // Linear2 dX (:573) + BAD-bwd (:576-578) in one tcgen05 kernel on the bf16 path (dA1 never
  // reaches HBM; db1 from its epilogue's column partials), else the contraction into dA1 and
  // the BAD-bwd kernel; Linear2 dW (:574); then the FFN half's column sums (dg2, dbe2, db2,
  // db1) in one launch
  const PhiloxKey pk_ffn = make_philox_key(cfg->p_ffn, cfg->seed, l4 + 2);
  {
    ReduceWs w = after(ffn_jobs[0]);
    w.defer = &ffn_jobs[1];
    WgemmArgs l2 = ffn_bwd_args(ctx, d, dtype, cfg, dY2, prm->W2, h, pk_ffn, dh, w.partials);
    if (bad_bytes_of(ctx, d, dtype)) l2.kb_in = (const uint8_t*)at(sv, SL.off[S_KBF]);
    const int R = wgemm_partial_rows(l2);
    if (wgemm_supported(l2) && (size_t)R * U <= w.cap_floats) {
      {
        OpTimer _t(ctx, ENC_OP_GEMM_L2_DX, st, 1);
        CK(launch_wgemm(l2, ctx->num_sms, st));
      }
      {
        cudaStream_t ss = fork(ENC_OP_GEMM_L2_DW);
        OpTimer _t(ctx, ENC_OP_GEMM_L2_DW, ss, 0);
        if ((r = wcontract(ctx, ENC_OP_GEMM_L2_DW, ss, dtype, F32, true, false, I, U, BJ, dY2, I, A1, U, 0.f,
                           g->dW2, U, nullptr, ss != st ? ctx->side_ws : nullptr)))
          return r;
      }
      // BAD-bwd has no launch of its own: db1's partials are finished with the half's
      // column sums (timed as ENC_OP_BAD_BWD only when that finalize launches here)
      CK(colsum_finish(w, R, U, U, g->db1, nullptr, nullptr, st));
      if (!ffn_deferred) {
        OpTimer _t(ctx, ENC_OP_BAD_BWD, st, 1);
        CK(launch_colsum_finalize_jobs(ffn_jobs, 2, st));
      }
    } else {
      {
        OpTimer _t(ctx, ENC_OP_GEMM_L2_DX, st, 0);
        if ((r = wcontract(ctx, ENC_OP_GEMM_L2_DX, st, dtype, dtype, false, false, BJ, U, I, dY2, I, prm->W2, U, 0.f,
                           dA1, U)))
          return r;
      }
      {
        cudaStream_t ss = fork(ENC_OP_GEMM_L2_DW);
        OpTimer _t(ctx, ENC_OP_GEMM_L2_DW, ss, 0);
        if ((r = wcontract(ctx, ENC_OP_GEMM_L2_DW, ss, dtype, F32, true, false, I, U, BJ, dY2, I, A1, U, 0.f,
                           g->dW2, U, nullptr, ss != st ? ctx->side_ws : nullptr)))
          return r;
      }
      OpTimer _t(ctx, ENC_OP_BAD_BWD, st, ffn_deferred ? 1 : 2);
      CK(launch_bad_bwd(dtype, B, J, U, dA1, h, nullptr, cfg->act, pk_ffn, boff, dh, g->db1, w,
                        st));
      if (!ffn_deferred) CK(launch_colsum_finalize_jobs(ffn_jobs, 2, st));
    }
  }
  // Linear1 dX (:579) accumulated onto dz2 (residual, paper `ebsb` :581), dW (:580)
  {
    OpTimer _t(ctx, ENC_OP_GEMM_L1_DX, st, 0);
    if ((r = wcontract(ctx, ENC_OP_GEMM_L1_DX, st, dtype, dtype, false, false, BJ, I, U, dh, U, prm->W1, I, 1.f, dX1,
                       I)))
      return r;
  }
  {
    cudaStream_t ss = fork(ENC_OP_GEMM_L1_DW);
    OpTimer _t(ctx, ENC_OP_GEMM_L1_DW, ss, 0);
    if ((r = wcontract(ctx, ENC_OP_GEMM_L1_DW, ss, dtype, F32, true, false, U, I, BJ, dh, U, X1, I, 0.f, g->dW1, I,
                       nullptr, ss != st ? ctx->side_ws : nullptr)))
      return r;
  }
  if (!(parts & 2)) CK(join());   // the FFN bucket is complete when the FFN part returns
  }  // FFN half
  if (!(parts & 2)) return ENC_OK;
  // BDRLN-bwd site 1 (:582-585): dz1 -> dX (residual to the layer input), dYo; its column
  // sums are finished with the QKV bias gradient at the end of the half
  ColsumJob att_jobs[4];
  {
    OpTimer _t(ctx, ENC_OP_BDRLN_BWD1, st, 1);
    ReduceWs w = ffn_deferred ? after(ffn_jobs[1]) : ws;
    w.defer = &att_jobs[0];
    CK(launch_bdrln_bwd(dtype, B, J, I, dX1, xh1, r1, prm->g1,
                        make_philox_key(cfg->p_hidden, cfg->seed, l4 + 1), boff, dX, dYo, g->dg1,
                        g->dbe1, g->dbo, w, st, (ctx->bdrln_variant >> 12) & 15,
                        ctx->mask_bytes ? (const uint8_t*)at(sv, SL.off[S_KB1]) : nullptr));
  }
  const ReduceWs wa = after(att_jobs[0]);   // the rest of the half reduces past those partials
  // Out dX (:586), dW (:587)
  {
    OpTimer _t(ctx, ENC_OP_GEMM_OUT_DX, st, 0);
    if ((r = wcontract(ctx, ENC_OP_GEMM_OUT_DX, st, dtype, dtype, false, false, BJ, I, I, dYo, I, prm->Wo, I, 0.f, dC,
                       I)))
      return r;
  }
  {
    cudaStream_t ss = fork(ENC_OP_GEMM_OUT_DW);
    OpTimer _t(ctx, ENC_OP_GEMM_OUT_DW, ss, 0);
    if ((r = wcontract(ctx, ENC_OP_GEMM_OUT_DW, ss, dtype, F32, true, false, I, I, BJ, dYo, I, C, I, 0.f, g->dWo, I,
                       nullptr, ss != st ? ctx->side_ws : nullptr)))
      return r;
  }
  // Gamma dX1 (:588): dA_bh = dC_bh V_bh^T;  Gamma dX2 (:589): dV_bh = A_bh^T dC_bh
  {
    OpTimer _t(ctx, ENC_OP_GEMM_AV_DA, st, fused_attn ? 0 : 1, !fused_attn);
    if (fused_attn) {
      // dA is produced inside the fused dA + BSB-bwd kernel below
    } else if (tc_attn) {
      CK(launch_attn_gemm(ENC_AG_DA, B, H, J, P, dC, I, V, ldqkv, dA, 0, st));
    } else {
      CK(launch_make_attn_ptrs(B, H, J, P, es, A, V, dC, dA, dV, ptr, st));
      CB(gemm_rm_batched(ctx->blas, dtype, false, true, J, K, P, 1.f,
                         (const void* const*)(ptr + 2 * BH), I, (const void* const*)(ptr + BH), P,
                         0.f, (void* const*)(ptr + 3 * BH), K, BH));
    }
  }
  // direct layout on the per-(b, h) kernels: AIB-bwd's bias gradient (:595) accumulates as
  // column sums in the dV / dQ / dK epilogues (partials [B*4][3I] in the reduction space)
  const bool bgrad_epi = direct && use_bh(ctx, J, P) && (size_t)B * 4 * 3 * I <= wa.cap_floats;
  float* bg = wa.partials;
  // fused + per-(b, h) path: the fused dA + BSB-bwd kernel is launched first and the dV
  // contraction (which needs only dC, P and the keep bits) on the side stream after it, so
  // dV's CTAs fill the SMs the fused kernel's uneven last wave leaves idle; joined before
  // the QKV contractions read dQKV
  const bool overlap = ctx->attn_overlap && ctx->side && fused_attn && use_bh(ctx, J, P);
  auto dv_step = [&](cudaStream_t sdv) -> int {
    OpTimer _t(ctx, ENC_OP_GEMM_AV_DV, sdv, tc_attn ? 1 : 0);
    if (fused_attn && use_bh(ctx, J, P))   // A was never stored: dropout on load from P
      CK(launch_attn_dv_bh(B, H, J, P, Pm, dC, I, dV, ldqkv, bgrad_epi ? bg + 2 * I : nullptr,
                           3 * I, (const uint32_t*)at(sv, SL.off[S_KB]),
                           make_philox_key(cfg->p_attn, cfg->seed, l4 + 0).scale, sdv));
    else if (bgrad_epi)
      CK(launch_attn_dv_bh(B, H, J, P, A, dC, I, dV, ldqkv, bg + 2 * I, 3 * I, nullptr, 1.f,
                           sdv));
    else if (tc_attn)
      CK(attn_contract(ctx, ENC_AG_DV, B, H, J, P, A, 0, dC, I, dV, ldqkv, sdv));
    else
      CB(gemm_rm_batched(ctx->blas, dtype, true, false, K, P, J, 1.f, (const void* const*)ptr, K,
                         (const void* const*)(ptr + 2 * BH), I, 0.f, (void* const*)(ptr + 4 * BH),
                         P, BH));
    return ENC_OK;
  };
  if (overlap) CK(cudaEventRecord(ctx->ev_fork, st));   // dC ready
  else if (int rr = dv_step(st)) return rr;
  // BSB-bwd (:590)
  {
    OpTimer _t(ctx, ENC_OP_BSB_BWD, st, 1);
    const bool dc_term = dc_term_of(ctx, fused_attn, J, P);
    if (fused_attn)  // Gamma dX1 (:588) + BSB-bwd (:590): dA stays in TMEM
      CK(launch_attn_da_bsbb(B, H, J, P, scale, dC, I, V, ldqkv, Pm,
                             make_philox_key(cfg->p_attn, cfg->seed, l4 + 0), boff,
                             (const uint32_t*)at(sv, SL.off[S_KB]), dS, st, overlap,
                             dc_term ? C : nullptr, dc_term ? at(sv, SL.off[S_CLO]) : nullptr,
                             I));
    else
      CK(launch_bsb_bwd(dtype, B, H, J, K, scale, dA, Pm,
                        make_philox_key(cfg->p_attn, cfg->seed, l4 + 0), boff, dS, st));
  }
  if (overlap) {
    CK(cudaStreamWaitEvent(ctx->side, ctx->ev_fork, 0));
    forked = true;
    if (int rr = dv_step(ctx->side)) return rr;
  }
  // QK^T dX1 (:591): dQ = dS K;  dX2 (:592): dK = dS^T Q
  const bool dqdk_one_pass = tc_attn && use_bh(ctx, J, P);
  {
    OpTimer _t(ctx, ENC_OP_GEMM_QK_DQ, st, tc_attn ? 1 : 0);
    if (dqdk_one_pass)   // dQ and dK from one read of dS
      CK(launch_attn_dqdk_bh(B, H, J, P, dS, Kt, ldqkv, Q, ldqkv, dQ, ldqkv, dK, ldqkv,
                             bgrad_epi ? bg : nullptr, bgrad_epi ? bg + I : nullptr, 3 * I, st));
    else if (tc_attn)
      CK(launch_attn_gemm(ENC_AG_DQ, B, H, J, P, dS, 0, Kt, ldqkv, dQ, ldqkv, st));
    else
      CB(gemm_rm_strided(ctx->blas, dtype, false, false, J, P, K, 1.f, dS, K, (long long)J * K, Kt,
                         P, (long long)K * P, 0.f, dQ, P, (long long)J * P, BH));
  }
  {
    OpTimer _t(ctx, ENC_OP_GEMM_QK_DK, st, tc_attn && !dqdk_one_pass ? 1 : 0, !dqdk_one_pass);
    if (dqdk_one_pass) {
      // computed with dQ above
    } else if (tc_attn)
      CK(launch_attn_gemm(ENC_AG_DK, B, H, J, P, dS, 0, Q, ldqkv, dK, ldqkv, st));
    else
      CB(gemm_rm_strided(ctx->blas, dtype, true, false, K, P, J, 1.f, dS, K, (long long)J * K, Q, P,
                         (long long)J * P, 0.f, dK, P, (long long)K * P, BH));
  }
  if (overlap) CK(join());   // dV (side stream) complete: dQKV and its bias partials whole
  // AIB-bwd (:595): the layout pass; on the direct path dQKV is already assembled and the
  // bias gradient rides in the QKV dW contraction's epilogue (or a column sum below)
  if (!direct) {
    OpTimer _t(ctx, ENC_OP_AIB_BWD, st, 2);
    CK(launch_aib_bwd(dtype, B, J, H, P, dQ, dK, dV, dQKV, g->dbqkv, wa, st));
  }
  // the attention half's column sums in one launch: BDRLN-bwd site 1 (dg1, dbe1, dbo), the
  // QKV bias gradient from the per-(b,h) epilogues' B*4 partial rows (and, for the whole
  // backward, the FFN half's).  Every input is final here: on the second side stream it
  // overlaps the Q,K,V contractions instead of following them
  auto finalize_att = [&](cudaStream_t fs) -> cudaError_t {
    int nj = 1;
    if (bgrad_epi) {
      att_jobs[1].partials = bg;
      att_jobs[1].R = B * 4;
      att_jobs[1].ncols = att_jobs[1].nper = 3 * I;
      att_jobs[1].out0 = g->dbqkv;
      nj = 2;
    }
    if (ffn_deferred) {
      att_jobs[nj++] = ffn_jobs[0];
      att_jobs[nj++] = ffn_jobs[1];
    }
    return launch_colsum_finalize_jobs(att_jobs, nj, fs);
  };
  const bool early_fin =
      (bgrad_epi || !direct) && ctx->side2 && (ctx->bwd_side == 2 || ctx->bwd_side == 3);
  bool forked2 = false;
  if (early_fin) {
    CK(cudaEventRecord(ctx->ev_fork2, st));
    CK(cudaStreamWaitEvent(ctx->side2, ctx->ev_fork2, 0));
    forked2 = true;
    OpTimer _t(ctx, bgrad_epi ? ENC_OP_AIB_BWD : ENC_OP_BDRLN_BWD1, ctx->side2, 1);
    CK(finalize_att(ctx->side2));
  }
  // Q,K,V dX (:593) accumulated onto dz1 (= BEI, :596), dW (:594)
  // (algebraic fusion, Table A.2: one dX / dW contraction per group of stacked blocks --
  // dX accumulates every group onto dz1, dW writes the group's rows of dWqkv)
  int ngrp = 0, gstart[3], gcount[3];
  qkv_groups(ctx->qkv_fusion_bwd, &ngrp, gstart, gcount);
  {
    OpTimer _t(ctx, ENC_OP_GEMM_QKV_DX, st, 0);
    for (int gi = 0; gi < ngrp; ++gi) {
      const int s0 = gstart[gi], nI = gcount[gi] * I;
      if ((r = wcontract(ctx, ENC_OP_GEMM_QKV_DX, st, dtype, dtype, false, false, BJ, I, nI,
                         (const char*)dQKV + (size_t)s0 * I * es, 3 * I,
                         (const char*)prm->Wqkv + (size_t)s0 * I * I * es, I, 1.f, dX, I)))
        return r;
    }
  }
  {
    cudaStream_t ss = fork(ENC_OP_GEMM_QKV_DW);
    OpTimer _t(ctx, ENC_OP_GEMM_QKV_DW, ss, 0);
    for (int gi = 0; gi < ngrp; ++gi) {
      const int s0 = gstart[gi], nI = gcount[gi] * I;
      if ((r = wcontract(ctx, ENC_OP_GEMM_QKV_DW, ss, dtype, F32, true, false, nI, I, BJ,
                         (const char*)dQKV + (size_t)s0 * I * es, 3 * I, X, I, 0.f,
                         g->dWqkv + (size_t)s0 * I * I, I, nullptr, ss != st ? ctx->side_ws : nullptr)))
        return r;
    }
  }
  if (direct && !bgrad_epi) {
    // bias gradient as a column sum of dQKV (cuBLASLt's BGRAD epilogue on the dW
    // contraction measured slower than this separate pass)
    OpTimer _t(ctx, ENC_OP_AIB_BWD, st, 2);
    CK(launch_colsum(dtype, BJ, 3 * I, dQKV, g->dbqkv, wa, st));
  }
  if (!early_fin) {
    OpTimer _t(ctx, bgrad_epi ? ENC_OP_AIB_BWD : ENC_OP_BDRLN_BWD1, st, 1);
    CK(finalize_att(st));
  }
  if (forked2) {
    CK(cudaEventRecord(ctx->ev_join2, ctx->side2));
    CK(cudaStreamWaitEvent(st, ctx->ev_join2, 0));
  }
  CK(join());
  return ENC_OK;
}

int encoder_layer_backward(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                           const enc_params* prm, const void* X, const void* saved,
                           const void* dY, void* dX, const enc_grads* g, void* scratch,
                           enc_stream_t stream) {
  return backward_impl(ctx, d, dtype, cfg, prm, X, saved, dY, dX, g, scratch, stream, 3);
}

int encoder_layer_backward_part(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                                const enc_params* prm, const void* X, const void* saved,
                                const void* dY, void* dX, const enc_grads* g, void* scratch,
                                int part, enc_stream_t stream) {
  if (part != ENC_BWD_FFN && part != ENC_BWD_ATTN) return ENC_EINVAL;
  return backward_impl(ctx, d, dtype, cfg, prm, X, saved, dY, dX, g, scratch, stream,
                       part == ENC_BWD_FFN ? 1 : 2);
}

int encoder_layer_step_host(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                            const enc_params* prm, const void* X_host, const void* dY_host,
                            void* Y_host, void* dX_host, void* X_dev, void* dY_dev, void* Y_dev,
                            void* dX_dev, const float* mask_bias, const enc_grads* g, void* saved,
                            void* scratch, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_dims(d, dtype);
  if (r) return r;
  if (!X_host || !dY_host || !Y_host || !dX_host) return ENC_ENULL;
  CHECK_PTRS(X_dev, dY_dev, Y_dev, dX_dev);
  cudaStream_t st = (cudaStream_t)stream;
  const size_t bytes = (size_t)d->B * d->J * d->I * esize(dtype);
  // X in on the layer stream; dY in on copy_in while the forward runs; Y out on copy_out
  // while the backward runs; dX out on the layer stream.  The call's stream finishes only
  // after every copy (it waits for copy_out at the end).
  CK(cudaEventRecord(ctx->ev_start, st));
  CK(cudaStreamWaitEvent(ctx->copy_in, ctx->ev_start, 0));
  CK(cudaMemcpyAsync(X_dev, X_host, bytes, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(dY_dev, dY_host, bytes, cudaMemcpyHostToDevice, ctx->copy_in));
  CK(cudaEventRecord(ctx->ev_in, ctx->copy_in));
  r = encoder_layer_forward(ctx, d, dtype, cfg, prm, X_dev, mask_bias, Y_dev, saved, scratch, stream);
  if (r) return r;
  CK(cudaEventRecord(ctx->ev_fwd, st));
  CK(cudaStreamWaitEvent(ctx->copy_out, ctx->ev_fwd, 0));
  CK(cudaMemcpyAsync(Y_host, Y_dev, bytes, cudaMemcpyDeviceToHost, ctx->copy_out));
  CK(cudaEventRecord(ctx->ev_out, ctx->copy_out));
  CK(cudaStreamWaitEvent(st, ctx->ev_in, 0));
  r = encoder_layer_backward(ctx, d, dtype, cfg, prm, X_dev, saved, dY_dev, dX_dev, g, scratch, stream);
  if (r) return r;
  CK(cudaMemcpyAsync(dX_host, dX_dev, bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamWaitEvent(st, ctx->ev_out, 0));
  return ENC_OK;
}

// input copies on copy_in, behind the work already on `st`, joined into `st`
static int prefetch(enc_ctx* ctx, size_t bytes, const void* X_host, const void* dY_host,
                    void* X_dev, void* dY_dev, cudaStream_t st) {
  CK(cudaEventRecord(ctx->ev_pfs, st));
  CK(cudaStreamWaitEvent(ctx->copy_in, ctx->ev_pfs, 0));
  CK(cudaMemcpyAsync(X_dev, X_host, bytes, cudaMemcpyHostToDevice, ctx->copy_in));
  CK(cudaMemcpyAsync(dY_dev, dY_host, bytes, cudaMemcpyHostToDevice, ctx->copy_in));
  CK(cudaEventRecord(ctx->ev_pf, ctx->copy_in));
  CK(cudaStreamWaitEvent(st, ctx->ev_pf, 0));
  return ENC_OK;
}

int enc_adamw_step(enc_ctx* ctx, int64_t n, float* master, float* m, float* v, const float* grad,
                   const enc_opt_segment* segs, int nseg, double lr, double beta1,
                   double beta2, double eps, double weight_decay, int step, double grad_scale,
                   enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  if (n < 0 || step < 1 || nseg < 1 || nseg > ENC_OPT_MAX_SEGMENTS || !(beta1 >= 0.0) ||
      !(beta1 < 1.0) || !(beta2 >= 0.0) || !(beta2 < 1.0))
    return ENC_EINVAL;
  if (n % 4) return ENC_EALIGN;
  if (!segs) return ENC_ENULL;
  CHECK_PTRS(master, m, v, grad);
  OptSeg s[kOptMaxSegs];
  int64_t at = 0;
  for (int k = 0; k < nseg; ++k) {
    const enc_opt_segment& e = segs[k];
    if (e.begin != at || e.n < 0) return ENC_EINVAL;
    if (e.begin % 4 || e.n % 4) return ENC_EALIGN;
    if (e.dtype != ENC_BF16 && e.dtype != ENC_FP32) return ENC_EDTYPE;
    if (e.n > 0) CHECK_PTRS(e.out);
    if (e.n > 0 && ((uintptr_t)e.out % (e.dtype == ENC_BF16 ? 8 : 16))) return ENC_EALIGN;
    if (e.no_decay != 0 && e.no_decay != 1) return ENC_EINVAL;
    s[k] = OptSeg{e.begin, e.n, e.out, e.dtype, e.no_decay};
    at += e.n;
  }
  if (at != n) return ENC_EINVAL;
  ctx->launches += n > 0;
  CK(launch_adamw(n, master, m, v, grad, s, nseg, lr, beta1, beta2, eps, weight_decay, step,
                  grad_scale, (cudaStream_t)stream));
  return ENC_OK;
}

int enc_prefetch_inputs(enc_ctx* ctx, const enc_dims* d, int dtype, const void* X_host,
                        const void* dY_host, void* X_dev, void* dY_dev, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_dims(d, dtype);
  if (r) return r;
  if (!X_host || !dY_host) return ENC_ENULL;
  CHECK_PTRS(X_dev, dY_dev);
  return prefetch(ctx, (size_t)d->B * d->J * d->I * esize(dtype), X_host, dY_host, X_dev, dY_dev,
                  (cudaStream_t)stream);
}

int encoder_layer_step_host_pipelined(enc_ctx* ctx, const enc_dims* d, int dtype,
                                      const enc_cfg* cfg, const enc_params* prm,
                                      const void* X_dev, const void* dY_dev, void* Y_dev,
                                      void* dX_dev, void* Y_host, const void* X_next_host,
                                      const void* dY_next_host, void* X_next_dev,
                                      void* dY_next_dev, const void* dX_prev_dev,
                                      void* dX_prev_host, const float* mask_bias,
                                      const enc_grads* g, void* saved, void* scratch,
                                      enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_dims(d, dtype);
  if (r) return r;
  if (!Y_host) return ENC_ENULL;
  CHECK_PTRS(X_dev, dY_dev, Y_dev, dX_dev);
  const size_t bytes = (size_t)d->B * d->J * d->I * esize(dtype);
  // buffers the copies touch while the layer runs must not overlap what the layer reads or
  // writes (byte ranges; the previous dX may BE this step's dX buffer, then the backward
  // waits for its copy)
  size_t sv_bytes = 0, sc_bytes = 0;
  if ((r = enc_layer_sizes(d, dtype, &sv_bytes, &sc_bytes))) return r;
  auto overlap = [](const void* a, size_t na, const void* b, size_t nb) {
    const char *pa = (const char*)a, *pb = (const char*)b;
    return a && b && pa < pb + nb && pb < pa + na;
  };
  const void* layer_bufs[6] = {X_dev, dY_dev, Y_dev, dX_dev, saved, scratch};
  const size_t layer_sz[6] = {bytes, bytes, bytes, bytes, sv_bytes, sc_bytes};
  const bool next = X_next_host != nullptr || dY_next_host != nullptr;
  if (next) {
    if (!X_next_host || !dY_next_host) return ENC_ENULL;
    CHECK_PTRS(X_next_dev, dY_next_dev);
    if (overlap(X_next_dev, bytes, dY_next_dev, bytes)) return ENC_EINVAL;
    for (int i = 0; i < 6; ++i)
      if (overlap(X_next_dev, bytes, layer_bufs[i], layer_sz[i]) ||
          overlap(dY_next_dev, bytes, layer_bufs[i], layer_sz[i]))
        return ENC_EINVAL;
  }
  const bool prev = dX_prev_dev != nullptr || dX_prev_host != nullptr;
  if (prev) {
    if (!dX_prev_host) return ENC_ENULL;
    CHECK_PTRS(dX_prev_dev);
    for (int i = 0; i < 6; ++i)
      if (i != 3 && overlap(dX_prev_dev, bytes, layer_bufs[i], layer_sz[i])) return ENC_EINVAL;
    if (overlap(dX_prev_dev, bytes, dX_dev, bytes) && dX_prev_dev != dX_dev) return ENC_EINVAL;
  }
  cudaStream_t st = (cudaStream_t)stream;
  // fork both copy streams here: the next step's inputs in (their buffers' last reader,
  // the previous step, is complete at this point of `st`), the previous step's dX out
  CK(cudaEventRecord(ctx->ev_pfs, st));
  if (next) {
    CK(cudaStreamWaitEvent(ctx->copy_in, ctx->ev_pfs, 0));
    CK(cudaMemcpyAsync(X_next_dev, X_next_host, bytes, cudaMemcpyHostToDevice, ctx->copy_in));
    CK(cudaMemcpyAsync(dY_next_dev, dY_next_host, bytes, cudaMemcpyHostToDevice, ctx->copy_in));
    CK(cudaEventRecord(ctx->ev_pf, ctx->copy_in));
  }
  CK(cudaStreamWaitEvent(ctx->copy_out, ctx->ev_pfs, 0));
  const bool dx_alias = prev && dX_prev_dev == dX_dev;
  if (prev) {
    CK(cudaMemcpyAsync(dX_prev_host, dX_prev_dev, bytes, cudaMemcpyDeviceToHost, ctx->copy_out));
    if (dx_alias) CK(cudaEventRecord(ctx->ev_out, ctx->copy_out));
  }
  // on an error after the fork, both copy streams are joined back into `st` before
  // returning (an active capture must not be left with unjoined work)
  auto join_copies = [&](int rc) {
    cudaEventRecord(ctx->ev_out, ctx->copy_out);
    cudaStreamWaitEvent(st, ctx->ev_out, 0);
    if (next) cudaStreamWaitEvent(st, ctx->ev_pf, 0);
    return rc;
  };
  r = encoder_layer_forward(ctx, d, dtype, cfg, prm, X_dev, mask_bias, Y_dev, saved, scratch,
                            stream);
  if (r) return join_copies(r);
  cudaError_t ce = cudaEventRecord(ctx->ev_fwd, st);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ctx->copy_out, ctx->ev_fwd, 0);
  if (ce == cudaSuccess)
    ce = cudaMemcpyAsync(Y_host, Y_dev, bytes, cudaMemcpyDeviceToHost, ctx->copy_out);
  // the previous step's dX in the same buffer: its copy finishes before the backward writes
  if (ce == cudaSuccess && dx_alias) ce = cudaStreamWaitEvent(st, ctx->ev_out, 0);
  if (ce != cudaSuccess) return join_copies(cuda_fail(ce));
  r = encoder_layer_backward(ctx, d, dtype, cfg, prm, X_dev, saved, dY_dev, dX_dev, g, scratch,
                             stream);
  if (r) return join_copies(r);
  // join: every copy this call issued is complete when `stream` passes its end
  CK(cudaEventRecord(ctx->ev_out, ctx->copy_out));
  CK(cudaStreamWaitEvent(st, ctx->ev_out, 0));
  if (next) CK(cudaStreamWaitEvent(st, ctx->ev_pf, 0));
  return ENC_OK;
}

}  // extern "C"

// ------------------------------------------------------------------ cross attention
// Encoder-decoder attention sublayer ("fuse keys and values in
// encoder/decoder attention"): queries from X [B,J,I], keys and values from the memory
// Mem [B,K,I] through ONE stacked contraction with [W^K; W^V] -> KV [B,K,2I], then the
// encoder layer's BSB (site 0, K keys) and BDRLN (site 1, residual X).  Q, K, V are read in
// place (row strides I and 2I) by the attention contractions: the tiled tcgen05 kernels
// when bf16, P = 64 and J, K are multiples of 128, else cuBLAS (strided over the heads of
// each batch element).
namespace {
enum XSaved { XS_Q, XS_KV, XS_P, XS_A, XS_C, XS_XH, XS_R, XS_N };
enum XFwd { XF_S, XF_YO, XF_N };
enum XBwd { XB_DYO, XB_DC, XB_DA, XB_DS, XB_DQ, XB_DKV, XB_N };
Layout xsaved_layout(const enc_dims* d, int dtype) {
  const size_t es = esize(dtype), BJ = (size_t)d->B * d->J, BK = (size_t)d->B * d->K;
  const size_t s = (size_t)d->B * d->H * d->J * d->K * es;
  const size_t sz[XS_N] = {BJ * d->I * es, BK * 2 * d->I * es, s, s, BJ * d->I * es,
                           BJ * d->I * es, BJ * sizeof(float)};
  return make_layout(sz, XS_N);
}
Layout xfwd_layout(const enc_dims* d, int dtype) {
  const size_t es = esize(dtype), BJ = (size_t)d->B * d->J;
  const size_t sz[XF_N] = {(size_t)d->B * d->H * d->J * d->K * es, BJ * d->I * es};
  return make_layout(sz, XF_N);
}
Layout xbwd_layout(const enc_dims* d, int dtype) {
  const size_t es = esize(dtype), BJ = (size_t)d->B * d->J, BK = (size_t)d->B * d->K;
  const size_t s = (size_t)d->B * d->H * d->J * d->K * es;
  const size_t sz[XB_N] = {BJ * d->I * es, BJ * d->I * es, s, s, BJ * d->I * es,
                           BK * 2 * d->I * es};
  return make_layout(sz, XB_N);
}
}  // namespace

static int check_xdims(const enc_dims* d, int dtype) {
  if (!d) return ENC_ENULL;
  if (!valid_dtype(dtype)) return ENC_EDTYPE;
  if (d->B < 0 || d->J <= 0 || d->K <= 0 || d->H <= 0 || d->P <= 0) return ENC_EINVAL;
  if (d->W != d->P || d->I != d->H * d->P) return ENC_EINVAL;
  if (d->I % 8 || d->K % 8 || d->P % 8) return ENC_EALIGN;
  if (!rowop_supported(d->K) || !rowop_supported(d->I) || !bdrln_bwd_supported(d->I, dtype))
    return ENC_EUNSUPPORTED;
  if ((int64_t)d->B * (d->J > d->K ? d->J : d->K) * 2 * d->I / 8 >= INT32_MAX ||
      (int64_t)d->B * d->H * d->J >= INT32_MAX)
    return ENC_EUNSUPPORTED;
  return ENC_OK;
}

// One attention contraction of the cross-attention sublayer (which = ENC_AG_*): X, Y, Z as
// in enc_attn_gemm, P-wide operands token-major with row strides ldx / ldy / ldz, [J x K]
// operands head-major [B,H,J,K].
static int xcontract(enc_ctx* ctx, int which, int dtype, int B, int H, int J, int K, int P,
                     const void* X, int64_t ldx, const void* Y, int64_t ldy, void* Z, int64_t ldz,
                     cudaStream_t st) {
  if (dtype == ENC_BF16 && ctx->attn_tc && P == 64 && J % 128 == 0 && K % 128 == 0) {
    CK(launch_attn_gemm(which, B, H, J, P, X, ldx, Y, ldy, Z, ldz, st, K));
    ctx->launches += 1;
    return ENC_OK;
  }
  const size_t es = esize(dtype);
  const long long jk = (long long)J * K;
  for (int b = 0; b < B; ++b) {
    auto tok = [&](const void* p, int rows, int64_t ld) {   // batch b of a token-major operand
      return (const char*)p + (size_t)b * rows * ld * es;
    };
    auto hm = [&](const void* p) { return (const char*)p + (size_t)b * H * jk * es; };
    cublasStatus_t s = CUBLAS_STATUS_SUCCESS;
    switch (which) {
      case ENC_AG_QK:   // S[J,K] = Q[J,P] K[K,P]^T
      case ENC_AG_DA:   // dA[J,K] = dC[J,P] V[K,P]^T
        s = gemm_rm_strided(ctx->blas, dtype, false, true, J, K, P, 1.f, tok(X, J, ldx), (int)ldx,
                            P, tok(Y, K, ldy), (int)ldy, P, 0.f, (void*)hm(Z), K, jk, H);
        break;
      case ENC_AG_AV:   // C[J,P] = A[J,K] V[K,P]
      case ENC_AG_DQ:   // dQ[J,P] = dS[J,K] K[K,P]
        s = gemm_rm_strided(ctx->blas, dtype, false, false, J, P, K, 1.f, hm(X), K, jk,
                            tok(Y, K, ldy), (int)ldy, P, 0.f, (void*)tok(Z, J, ldz), (int)ldz, P,
                            H);
        break;
      case ENC_AG_DV:   // dV[K,P] = A[J,K]^T dC[J,P]
      case ENC_AG_DK:   // dK[K,P] = dS[J,K]^T Q[J,P]
        s = gemm_rm_strided(ctx->blas, dtype, true, false, K, P, J, 1.f, hm(X), K, jk,
                            tok(Y, J, ldy), (int)ldy, P, 0.f, (void*)tok(Z, K, ldz), (int)ldz, P,
                            H);
        break;
      default:
        return ENC_EINVAL;
    }
    if (s != CUBLAS_STATUS_SUCCESS) return ENC_ECUBLAS;
  }
  return ENC_OK;
}

// C[rows, N] = A W^T + bias, the bias in the contraction epilogue where available, else a
// row-bias pass
static int linear_bias(enc_ctx* ctx, int op, cudaStream_t st, int dtype, int rows, int N, int Kd,
                       const void* A, const void* W, const float* bias, void* C) {
  int r = wcontract(ctx, op, st, dtype, dtype, false, true, rows, N, Kd, A, Kd, W, Kd, 0.f, C, N,
                    bias);
  if (r == ENC_OK) return ENC_OK;
  if (r != ENC_EUNSUPPORTED) return r;
  if ((r = wcontract(ctx, op, st, dtype, dtype, false, true, rows, N, Kd, A, Kd, W, Kd, 0.f, C,
                     N)))
    return r;
  CK(launch_bias_rows(dtype, rows, N, C, bias, st));
  ctx->launches += 1;
  return ENC_OK;
}

extern "C" {

int enc_xattn_sizes(const enc_dims* d, int dtype, size_t* saved_bytes, size_t* scratch_bytes) {
  int r = check_xdims(d, dtype);
  if (r) return r;
  if (saved_bytes) *saved_bytes = xsaved_layout(d, dtype).total;
  if (scratch_bytes) {
    const size_t f = xfwd_layout(d, dtype).total, b = xbwd_layout(d, dtype).total;
    *scratch_bytes = f > b ? f : b;
  }
  return ENC_OK;
}

static int check_xparams(const enc_xattn_params* p) {
  if (!p) return ENC_ENULL;
  CHECK_PTRS(p->Wq, p->Wkv, p->Wo, p->bq, p->bkv, p->bo, p->g, p->be);
  return ENC_OK;
}

int enc_xattn_forward(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                      const enc_xattn_params* prm, const void* X, const void* Mem,
                      const float* mask_bias, void* Y, void* saved, void* scratch,
                      enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_xdims(d, dtype);
  if (r) return r;
  if ((r = check_cfg(cfg))) return r;
  if (cfg->causal) return ENC_EINVAL;   // causal masking needs J == K (self-attention)
  if ((r = check_xparams(prm))) return r;
  CHECK_PTRS(X, Mem, Y, saved, scratch);
  if (mask_bias && !aligned16(mask_bias)) return ENC_EALIGN;
  if (d->B == 0) return ENC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  CB(cublasSetStream(ctx->blas, st));
  const int B = d->B, J = d->J, K = d->K, H = d->H, P = d->P, I = d->I;
  const Layout SL = xsaved_layout(d, dtype), FL = xfwd_layout(d, dtype);
  void *Q = at(saved, SL.off[XS_Q]), *KV = at(saved, SL.off[XS_KV]);
  void *Pm = at(saved, SL.off[XS_P]), *A = at(saved, SL.off[XS_A]), *C = at(saved, SL.off[XS_C]);
  void* xh = at(saved, SL.off[XS_XH]);
  float* rs = (float*)at(saved, SL.off[XS_R]);
  void *S = at(scratch, FL.off[XF_S]), *Yo = at(scratch, FL.off[XF_YO]);
  const size_t es = esize(dtype);
  const uint64_t l4 = 4ull * cfg->layer_id;
  const float scale = 1.0f / sqrtf((float)P);
  // Q = X Wq^T + bq;  [K | V] = Mem [Wk; Wv]^T + bkv (one stacked contraction)
  if ((r = linear_bias(ctx, ENC_OP_GEMM_QKV, st, dtype, B * J, I, I, X, prm->Wq, prm->bq, Q)))
    return r;
  if ((r = linear_bias(ctx, ENC_OP_GEMM_QKV, st, dtype, B * K, 2 * I, I, Mem, prm->Wkv, prm->bkv,
                       KV)))
    return r;
  // S = Q K^T per (b, h), BSB (site 0), C = A V
  if ((r = xcontract(ctx, ENC_AG_QK, dtype, B, H, J, K, P, Q, I, KV, 2 * I, S, 0, st))) return r;
  CK(launch_bsb_fwd(dtype, B, H, J, K, scale, S, mask_bias,
                    make_philox_key(cfg->p_attn, cfg->seed, l4 + 0), cfg->batch_offset, Pm, A, st));
  ctx->launches += 1;
  if ((r = xcontract(ctx, ENC_AG_AV, dtype, B, H, J, K, P, A, 0, (char*)KV + (size_t)I * es,
                     2 * I, C, I, st)))
    return r;
  // Out, BDRLN (site 1) with the residual X
  if ((r = wcontract(ctx, ENC_OP_GEMM_OUT, st, dtype, dtype, false, true, B * J, I, I, C, I,
                     prm->Wo, I, 0.f, Yo, I)))
    return r;
  CK(launch_bdrln_fwd(dtype, B, J, I, Yo, prm->bo, X, prm->g, prm->be, cfg->ln_eps,
                      make_philox_key(cfg->p_hidden, cfg->seed, l4 + 1), cfg->batch_offset, Y, xh,
                      rs, st));
  ctx->launches += 1;
  return ENC_OK;
}

int enc_xattn_backward(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                       const enc_xattn_params* prm, const void* X, const void* Mem,
                       const void* saved, const void* dY, void* dX, void* dMem,
                       const enc_xattn_grads* g, void* scratch, enc_stream_t stream) {
  if (!ctx) return ENC_ENULL;
  int r = check_xdims(d, dtype);
  if (r) return r;
  if ((r = check_cfg(cfg))) return r;
  if (cfg->causal) return ENC_EINVAL;
  if ((r = check_xparams(prm))) return r;
  if (!g) return ENC_ENULL;
  CHECK_PTRS(X, Mem, saved, dY, dX, dMem, scratch, g->dWq, g->dWkv, g->dWo, g->dbq, g->dbkv,
             g->dbo, g->dg, g->dbe);
  cudaStream_t st = (cudaStream_t)stream;
  const int B = d->B, J = d->J, K = d->K, H = d->H, P = d->P, I = d->I;
  if (B == 0) {
    const size_t n[8] = {(size_t)I * I, (size_t)2 * I * I, (size_t)I * I, (size_t)I,
                         (size_t)2 * I, (size_t)I, (size_t)I, (size_t)I};
    float* p[8] = {g->dWq, g->dWkv, g->dWo, g->dbq, g->dbkv, g->dbo, g->dg, g->dbe};
    for (int i = 0; i < 8; ++i) CK(cudaMemsetAsync(p[i], 0, n[i] * sizeof(float), st));
    return ENC_OK;
  }
  CB(cublasSetStream(ctx->blas, st));
  const size_t es = esize(dtype);
  const Layout SL = xsaved_layout(d, dtype), BL = xbwd_layout(d, dtype);
  void* sv = (void*)saved;
  void *Q = at(sv, SL.off[XS_Q]), *KV = at(sv, SL.off[XS_KV]);
  void *Pm = at(sv, SL.off[XS_P]), *A = at(sv, SL.off[XS_A]), *C = at(sv, SL.off[XS_C]);
  void* xh = at(sv, SL.off[XS_XH]);
  float* rs = (float*)at(sv, SL.off[XS_R]);
  void *dYo = at(scratch, BL.off[XB_DYO]), *dC = at(scratch, BL.off[XB_DC]);
  void *dA = at(scratch, BL.off[XB_DA]), *dS = at(scratch, BL.off[XB_DS]);
  void *dQ = at(scratch, BL.off[XB_DQ]), *dKV = at(scratch, BL.off[XB_DKV]);
  const uint64_t l4 = 4ull * cfg->layer_id;
  const float scale = 1.0f / sqrtf((float)P);
  const ReduceWs ws = ws_of(ctx);
  const int F32 = ENC_FP32;
  // BDRLN-bwd (site 1): dz -> dX (residual), dYo; dg, dbe, dbo
  CK(launch_bdrln_bwd(dtype, B, J, I, dY, xh, rs, prm->g,
                      make_philox_key(cfg->p_hidden, cfg->seed, l4 + 1), cfg->batch_offset, dX,
                      dYo, g->dg, g->dbe, g->dbo, ws, st));
  ctx->launches += 2;
  // Out dX, dW
  if ((r = wcontract(ctx, ENC_OP_GEMM_OUT_DX, st, dtype, dtype, false, false, B * J, I, I, dYo, I,
                     prm->Wo, I, 0.f, dC, I)))
    return r;
  if ((r = wcontract(ctx, ENC_OP_GEMM_OUT_DW, st, dtype, F32, true, false, I, I, B * J, dYo, I, C,
                     I, 0.f, g->dWo, I)))
    return r;
  // dA = dC V^T, dV = A^T dC (into the V half of dKV), BSB-bwd, dQ = dS K, dK = dS^T Q
  char* V = (char*)KV + (size_t)I * es;
  if ((r = xcontract(ctx, ENC_AG_DA, dtype, B, H, J, K, P, dC, I, V, 2 * I, dA, 0, st))) return r;
  if ((r = xcontract(ctx, ENC_AG_DV, dtype, B, H, J, K, P, A, 0, dC, I,
                     (char*)dKV + (size_t)I * es, 2 * I, st)))
    return r;
  CK(launch_bsb_bwd(dtype, B, H, J, K, scale, dA, Pm,
                    make_philox_key(cfg->p_attn, cfg->seed, l4 + 0), cfg->batch_offset, dS, st));
  ctx->launches += 1;
  if ((r = xcontract(ctx, ENC_AG_DQ, dtype, B, H, J, K, P, dS, 0, KV, 2 * I, dQ, I, st))) return r;
  if ((r = xcontract(ctx, ENC_AG_DK, dtype, B, H, J, K, P, dS, 0, Q, I, dKV, 2 * I, st))) return r;
  // bias gradients (column sums), then dX += dQ Wq (beta = 1 onto dz), dMem = dKV [Wk; Wv]
  CK(launch_colsum(dtype, B * J, I, dQ, g->dbq, ws, st));
  CK(launch_colsum(dtype, B * K, 2 * I, dKV, g->dbkv, ws, st));
  ctx->launches += 4;
  if ((r = wcontract(ctx, ENC_OP_GEMM_QKV_DX, st, dtype, dtype, false, false, B * J, I, I, dQ, I,
                     prm->Wq, I, 1.f, dX, I)))
    return r;
  if ((r = wcontract(ctx, ENC_OP_GEMM_QKV_DX, st, dtype, dtype, false, false, B * K, I, 2 * I, dKV,
                     2 * I, prm->Wkv, I, 0.f, dMem, I)))
    return r;
  if ((r = wcontract(ctx, ENC_OP_GEMM_QKV_DW, st, dtype, F32, true, false, I, I, B * J, dQ, I, X,
                     I, 0.f, g->dWq, I)))
    return r;
  if ((r = wcontract(ctx, ENC_OP_GEMM_QKV_DW, st, dtype, F32, true, false, 2 * I, I, B * K, dKV,
                     2 * I, Mem, I, 0.f, g->dWkv, I)))
    return r;
  return ENC_OK;
}

}  // extern "C"
