// Weight contractions through cuBLASLt with per-shape algorithm selection by measurement —
// the paper's contraction tuning step (§5.1: "we benchmark ... every
// algorithm", best algorithm vs cuBLAS's heuristic up to 14.24% faster on V100, Fig. 3).
// For each (shape, layout, dtypes, epilogue) the first eager call times up to kMaxAlgos
// heuristic candidates on the caller's stream and caches the fastest; calls made while the
// stream is being captured into a CUDA graph use the cached choice (or the heuristic's first
// candidate when none has been measured).  Epilogues: none, +bias (fp32 bias over output
// columns), and the bias gradient of the second operand (column sums over the reduction
// dimension), which lets a weight-gradient GEMM also produce a bias gradient.
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <tuple>

#include "gemm.h"

namespace enc {

namespace {
constexpr int kMaxAlgos = 32;

cudaDataType_t dt(int dtype) { return dtype == 0 ? CUDA_R_16BF : CUDA_R_32F; }

using Key = std::tuple<int, int, int, int, int, int, int, int, int, int, int, int>;

struct Plan {
  cublasLtMatmulAlgo_t algo;
  bool tuned = false;
  bool valid = false;
};
}  // namespace

struct LtCtx {
  cublasLtHandle_t h = nullptr;
  void* ws = nullptr;
  size_t ws_bytes = 0;
  void* tmp = nullptr;         // output sink for timing runs (never the caller's buffers)
  size_t tmp_bytes = 0;
  std::map<Key, Plan> plans;
  std::mutex mu;
  int autotune = 0;   // measuring is opt-in (ENC_OPT_GEMM_AUTOTUNE): it allocates and syncs
};

LtCtx* lt_create(void* ws, size_t ws_bytes) {
  LtCtx* c = new LtCtx();
  if (cublasLtCreate(&c->h) != CUBLAS_STATUS_SUCCESS) {
    delete c;
    return nullptr;
  }
  c->ws = ws;
  c->ws_bytes = ws_bytes;
  return c;
}

void lt_destroy(LtCtx* c) {
  if (!c) return;
  if (c->h) cublasLtDestroy(c->h);
  if (c->tmp) cudaFree(c->tmp);
  delete c;
}

void lt_set_autotune(LtCtx* c, int on) { c->autotune = on; }

namespace {
struct Desc {
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t a = nullptr, b = nullptr, c = nullptr;
  ~Desc() {
    if (op) cublasLtMatmulDescDestroy(op);
    if (a) cublasLtMatrixLayoutDestroy(a);
    if (b) cublasLtMatrixLayoutDestroy(b);
    if (c) cublasLtMatrixLayoutDestroy(c);
  }
};
}  // namespace

// Row-major C[M,N] = op(A) op(B) (+ beta C) (+ epilogue); see gemm.cu for the operand swap.
cublasStatus_t lt_gemm_rm(LtCtx* L, int in_dtype, int out_dtype, bool tA, bool tB, int M, int N,
                          int K, const void* A, int lda, const void* B, int ldb, float beta,
                          void* C, int ldc, int epi, void* bias, cudaStream_t st, void* ws_override) {
  void* const ws = ws_override ? ws_override : L->ws;
  const cublasComputeType_t ct = in_dtype == 0 ? CUBLAS_COMPUTE_32F : CUBLAS_COMPUTE_32F_PEDANTIC;
  Desc d;
  cublasStatus_t s = cublasLtMatmulDescCreate(&d.op, ct, CUDA_R_32F);
  if (s) return s;
  const cublasOperation_t opA = tB ? CUBLAS_OP_T : CUBLAS_OP_N;  // Lt "A" = our B
  const cublasOperation_t opB = tA ? CUBLAS_OP_T : CUBLAS_OP_N;  // Lt "B" = our A
  cublasLtMatmulDescSetAttribute(d.op, CUBLASLT_MATMUL_DESC_TRANSA, &opA, sizeof(opA));
  cublasLtMatmulDescSetAttribute(d.op, CUBLASLT_MATMUL_DESC_TRANSB, &opB, sizeof(opB));
  cublasLtEpilogue_t e = CUBLASLT_EPILOGUE_DEFAULT;
  if (epi == LT_EPI_BIAS) e = CUBLASLT_EPILOGUE_BIAS;
  // our A is cuBLASLt's B: its bias gradient (length M = columns of D^T) is BGRADB
  if (epi == LT_EPI_BGRAD_A) e = CUBLASLT_EPILOGUE_BGRADB;
  cublasLtMatmulDescSetAttribute(d.op, CUBLASLT_MATMUL_DESC_EPILOGUE, &e, sizeof(e));
  if (epi != LT_EPI_NONE) {
    cublasLtMatmulDescSetAttribute(d.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias));
    // cuBLASLt accepts an fp32 bias only with an fp32 output: a bf16 output takes its bias
    // in bf16 (the caller passes a bf16 vector then); bias gradients are fp32
    const cudaDataType_t bt =
        epi == LT_EPI_BIAS && out_dtype == 0 ? CUDA_R_16BF : CUDA_R_32F;
    cublasLtMatmulDescSetAttribute(d.op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bt, sizeof(bt));
  }
  // column-major views (see gemm.cu): Lt A = our B, Lt B = our A, D = C^T [N x M]
  if ((s = cublasLtMatrixLayoutCreate(&d.a, dt(in_dtype), tB ? K : N, tB ? N : K, ldb))) return s;
  if ((s = cublasLtMatrixLayoutCreate(&d.b, dt(in_dtype), tA ? M : K, tA ? K : M, lda))) return s;
  if ((s = cublasLtMatrixLayoutCreate(&d.c, dt(out_dtype), N, M, ldc))) return s;
  const float alpha = 1.f;

  const Key key{in_dtype, out_dtype, tA, tB, M, N, K, lda, ldb, ldc, beta != 0.f, epi};
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cs);
  const bool capturing = cs != cudaStreamCaptureStatusNone;

  Plan plan;
  {
    std::lock_guard<std::mutex> g(L->mu);
    auto it = L->plans.find(key);
    if (it != L->plans.end()) plan = it->second;
  }
  if (!plan.valid || (!plan.tuned && !capturing && L->autotune)) {
    cublasLtMatmulPreference_t pref = nullptr;
    cublasLtMatmulPreferenceCreate(&pref);
    cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES,
                                         &L->ws_bytes, sizeof(L->ws_bytes));
    cublasLtMatmulHeuristicResult_t res[kMaxAlgos];
    int n = 0;
    s = cublasLtMatmulAlgoGetHeuristic(L->h, d.op, d.a, d.b, d.c, d.c, pref, kMaxAlgos, res, &n);
    cublasLtMatmulPreferenceDestroy(pref);
    if (s != CUBLAS_STATUS_SUCCESS || n == 0) return s ? s : CUBLAS_STATUS_NOT_SUPPORTED;
    plan.algo = res[0].algo;
    plan.valid = true;
    if (!capturing && L->autotune && n > 1) {
      // measure every candidate on a private output (and, for beta != 0, a private input)
      const size_t out_bytes = (size_t)M * ldc * (out_dtype == 0 ? 2 : 4);
      if (L->tmp_bytes < out_bytes) {
        if (L->tmp) cudaFree(L->tmp);
        L->tmp = nullptr;
        L->tmp_bytes = 0;
        if (cudaMalloc(&L->tmp, out_bytes) == cudaSuccess) L->tmp_bytes = out_bytes;
      }
      float* bsink = nullptr;
      if (epi != LT_EPI_NONE) cudaMalloc(&bsink, sizeof(float) * (size_t)(M > N ? M : N));
      if (L->tmp && (epi == LT_EPI_NONE || bsink)) {
        if (epi != LT_EPI_NONE)
          cublasLtMatmulDescSetAttribute(d.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bsink,
                                         sizeof(bsink));
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        float best = 1e30f;
        for (int i = 0; i < n; ++i) {
          if (res[i].state != CUBLAS_STATUS_SUCCESS) continue;
          bool ok = true;
          for (int w = 0; w < 2 && ok; ++w)   // warm-up
            ok = cublasLtMatmul(L->h, d.op, &alpha, B, d.a, A, d.b, &beta, L->tmp, d.c, L->tmp,
                                d.c, &res[i].algo, ws, L->ws_bytes, st) == CUBLAS_STATUS_SUCCESS;
          if (!ok) continue;
          cudaEventRecord(e0, st);
          for (int r = 0; r < 5; ++r)
            cublasLtMatmul(L->h, d.op, &alpha, B, d.a, A, d.b, &beta, L->tmp, d.c, L->tmp, d.c,
                           &res[i].algo, ws, L->ws_bytes, st);
          cudaEventRecord(e1, st);
          cudaEventSynchronize(e1);
          float ms = 0.f;
          cudaEventElapsedTime(&ms, e0, e1);
          if (ms < best) {
            best = ms;
            plan.algo = res[i].algo;
          }
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        plan.tuned = true;
        if (epi != LT_EPI_NONE)
          cublasLtMatmulDescSetAttribute(d.op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias,
                                         sizeof(bias));
      }
      if (bsink) cudaFree(bsink);
    }
    std::lock_guard<std::mutex> g(L->mu);
    L->plans[key] = plan;
  }
  return cublasLtMatmul(L->h, d.op, &alpha, B, d.a, A, d.b, &beta, C, d.c, C, d.c, &plan.algo,
                        ws, L->ws_bytes, st);
}

}  // namespace enc
