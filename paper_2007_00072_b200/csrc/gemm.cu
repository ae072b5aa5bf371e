// Contractions of the layer (Table A.1 tensor-contraction rows) through
// cuBLAS (tcgen05 tensor cores underneath on sm_100a).  The paper maps every einsum to a
// (batched) MMM and calls cublasGemmEx ("Tensor Contractions"); this
// file is the row-major wrapper the layer uses.  bf16 operands accumulate in fp32
// (PAPER.md:528 mixed precision); the fp32 path uses CUBLAS_COMPUTE_32F_PEDANTIC so TF32
// is never used (R13).
#include <cublas_v2.h>

#include "gemm.h"

namespace enc {

static cudaDataType_t dt(int dtype) { return dtype == 0 ? CUDA_R_16BF : CUDA_R_32F; }
static cublasComputeType_t ct(int dtype) {
  return dtype == 0 ? CUBLAS_COMPUTE_32F : CUBLAS_COMPUTE_32F_PEDANTIC;
}
static cublasOperation_t op(bool t) { return t ? CUBLAS_OP_T : CUBLAS_OP_N; }

// Row-major C[M,N] = alpha * op(A)[M,K] op(B)[K,N] + beta * C.  cuBLAS is column-major,
// so we compute C^T = op(B)^T op(A)^T: swap operands and M/N; a row-major matrix with
// leading dimension ld is its transpose in column-major with the same ld.
cublasStatus_t gemm_rm(cublasHandle_t h, int in_dtype, int out_dtype, bool tA, bool tB, int M,
                       int N, int K, float alpha, const void* A, int lda, const void* B,
                       int ldb, float beta, void* C, int ldc) {
  return cublasGemmEx(h, op(tB), op(tA), N, M, K, &alpha, B, dt(in_dtype), ldb, A,
                      dt(in_dtype), lda, &beta, C, dt(out_dtype), ldc, ct(in_dtype),
                      CUBLAS_GEMM_DEFAULT);
}

cublasStatus_t gemm_rm_strided(cublasHandle_t h, int dtype, bool tA, bool tB, int M, int N,
                               int K, float alpha, const void* A, int lda, long long sA,
                               const void* B, int ldb, long long sB, float beta, void* C,
                               int ldc, long long sC, int batch) {
  return cublasGemmStridedBatchedEx(h, op(tB), op(tA), N, M, K, &alpha, B, dt(dtype), ldb, sB,
                                    A, dt(dtype), lda, sA, &beta, C, dt(dtype), ldc, sC, batch,
                                    ct(dtype), CUBLAS_GEMM_DEFAULT);
}

cublasStatus_t gemm_rm_batched(cublasHandle_t h, int dtype, bool tA, bool tB, int M, int N,
                               int K, float alpha, const void* const* A, int lda,
                               const void* const* B, int ldb, float beta, void* const* C,
                               int ldc, int batch) {
  return cublasGemmBatchedEx(h, op(tB), op(tA), N, M, K, &alpha, B, dt(dtype), ldb, A,
                             dt(dtype), lda, &beta, C, dt(dtype), ldc, batch, ct(dtype),
                             CUBLAS_GEMM_DEFAULT);
}

}  // namespace enc
