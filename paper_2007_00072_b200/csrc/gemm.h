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
}  // namespace enc
