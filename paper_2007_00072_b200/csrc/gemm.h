#pragma once
#include <cublas_v2.h>

namespace enc {
cublasStatus_t gemm_rm(cublasHandle_t h, int in_dtype, int out_dtype, bool tA, bool tB, int M,
                       int N, int K, float alpha, const void* A, int lda, const void* B,
                       int ldb, float beta, void* C, int ldc);
cublasStatus_t gemm_rm_strided(cublasHandle_t h, int dtype, bool tA, bool tB, int M, int N,
                               int K, float alpha, const void* A, int lda, long long sA,
                               const void* B, int ldb, long long sB, float beta, void* C,
                               int ldc, long long sC, int batch);
cublasStatus_t gemm_rm_batched(cublasHandle_t h, int dtype, bool tA, bool tB, int M, int N,
                               int K, float alpha, const void* const* A, int lda,
                               const void* const* B, int ldb, float beta, void* const* C,
                               int ldc, int batch);

// cuBLASLt path with measured algorithm selection (gemm_lt.cu)
struct LtCtx;
enum { LT_EPI_NONE = 0, LT_EPI_BIAS = 1, LT_EPI_BGRAD_A = 2 };
LtCtx* lt_create(void* workspace, size_t workspace_bytes);
void lt_destroy(LtCtx* c);
void lt_set_autotune(LtCtx* c, int on);
// Row-major C[M,N] = op(A) op(B) + beta C; epi: LT_EPI_BIAS adds bias[N] to every row (bias in
// the output type: bf16 for a bf16 output, fp32 for fp32);
// LT_EPI_BGRAD_A also writes bias[M] = sum over K of op(A) (fp32 column sums of the
// reduction dimension).
cublasStatus_t lt_gemm_rm(LtCtx* L, int in_dtype, int out_dtype, bool tA, bool tB, int M, int N,
                          int K, const void* A, int lda, const void* B, int ldb, float beta,
                          void* C, int ldc, int epi, void* bias, cudaStream_t st,
                          void* ws_override = nullptr);
}  // namespace enc
