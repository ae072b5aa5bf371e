// Which cuBLASLt epilogues does this cuBLAS support for the encoder's QKV contractions?
// Row-major C[M,N] = op(A) op(B) expressed as column-major D^T (as in gemm_lt.cu):
//   fwd  QKV = X Wqkv^T + bias          (M = BJ, N = 3I, K = I), bf16 out, BIAS epilogue
//   bwd  dWqkv = dQKV^T X, dbqkv = colsum(dQKV)  (M = 3I, N = I, K = BJ), fp32 out, BGRADB
// Build: nvcc -O2 -o tools/lt_epi_probe tools/lt_epi_probe.cu -lcublasLt
#include <cublasLt.h>
#include <cuda_runtime.h>
#include <stdio.h>

static void probe(cublasLtHandle_t h, const char* name, cudaDataType_t dt_out, bool tA, bool tB,
                  int M, int N, int K, int lda, int ldb, int ldc, cublasLtEpilogue_t epi,
                  cudaDataType_t bias_t, bool set_bias_type) {
  cublasLtMatmulDesc_t op;
  cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F);
  const cublasOperation_t opA = tB ? CUBLAS_OP_T : CUBLAS_OP_N;
  const cublasOperation_t opB = tA ? CUBLAS_OP_T : CUBLAS_OP_N;
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &opA, sizeof(opA));
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &opB, sizeof(opB));
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_EPILOGUE, &epi, sizeof(epi));
  void* bias = nullptr;
  cudaMalloc(&bias, 4 * 65536);
  cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_POINTER, &bias, sizeof(bias));
  if (set_bias_type)
    cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_BIAS_DATA_TYPE, &bias_t,
                                   sizeof(bias_t));
  cublasLtMatrixLayout_t a, b, c;
  cublasLtMatrixLayoutCreate(&a, CUDA_R_16BF, tB ? K : N, tB ? N : K, ldb);
  cublasLtMatrixLayoutCreate(&b, CUDA_R_16BF, tA ? M : K, tA ? K : M, lda);
  cublasLtMatrixLayoutCreate(&c, dt_out, N, M, ldc);
  cublasLtMatmulPreference_t pref;
  cublasLtMatmulPreferenceCreate(&pref);
  size_t ws = 32u << 20;
  cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES, &ws,
                                       sizeof(ws));
  cublasLtMatmulHeuristicResult_t res[8];
  int n = 0;
  cublasStatus_t s = cublasLtMatmulAlgoGetHeuristic(h, op, a, b, c, c, pref, 8, res, &n);
  printf("%-48s status %2d  algos %d\n", name, (int)s, n);
  cublasLtMatmulPreferenceDestroy(pref);
  cublasLtMatrixLayoutDestroy(a);
  cublasLtMatrixLayoutDestroy(b);
  cublasLtMatrixLayoutDestroy(c);
  cublasLtMatmulDescDestroy(op);
  cudaFree(bias);
}

int main() {
  cublasLtHandle_t h;
  cublasLtCreate(&h);
  const int BJ = 4096, I = 1024;
  // forward QKV: row-major C[BJ,3I] = X[BJ,I] Wqkv[3I,I]^T  (tA = false, tB = true)
  probe(h, "fwd BIAS bf16 out, bias fp32", CUDA_R_16BF, false, true, BJ, 3 * I, I, I, I, 3 * I,
        CUBLASLT_EPILOGUE_BIAS, CUDA_R_32F, true);
  probe(h, "fwd BIAS bf16 out, bias default type", CUDA_R_16BF, false, true, BJ, 3 * I, I, I, I,
        3 * I, CUBLASLT_EPILOGUE_BIAS, CUDA_R_32F, false);
  probe(h, "fwd BIAS bf16 out, bias bf16", CUDA_R_16BF, false, true, BJ, 3 * I, I, I, I, 3 * I,
        CUBLASLT_EPILOGUE_BIAS, CUDA_R_16BF, true);
  probe(h, "fwd DEFAULT", CUDA_R_16BF, false, true, BJ, 3 * I, I, I, I, 3 * I,
        CUBLASLT_EPILOGUE_DEFAULT, CUDA_R_32F, false);
  // backward dWqkv: row-major C[3I,I] = dQKV[BJ,3I]^T X[BJ,I]  (tA = true, tB = false)
  probe(h, "bwd BGRADB fp32 out, bias fp32", CUDA_R_32F, true, false, 3 * I, I, BJ, 3 * I, I, I,
        CUBLASLT_EPILOGUE_BGRADB, CUDA_R_32F, true);
  probe(h, "bwd BGRADB fp32 out, bias default", CUDA_R_32F, true, false, 3 * I, I, BJ, 3 * I, I,
        I, CUBLASLT_EPILOGUE_BGRADB, CUDA_R_32F, false);
  probe(h, "bwd BGRADB bf16 out, bias fp32", CUDA_R_16BF, true, false, 3 * I, I, BJ, 3 * I, I, I,
        CUBLASLT_EPILOGUE_BGRADB, CUDA_R_32F, true);
  probe(h, "bwd BGRADA fp32 out (other operand)", CUDA_R_32F, true, false, 3 * I, I, BJ, 3 * I,
        I, I, CUBLASLT_EPILOGUE_BGRADA, CUDA_R_32F, true);
  // alternative: dWqkv^T = X^T dQKV  (row-major C[I,3I], tA = true, tB = false): bias grad of
  // our B operand = Lt A -> BGRADA
  probe(h, "bwd' C[I,3I]=X^T dQKV, BGRADA fp32 out", CUDA_R_32F, true, false, I, 3 * I, BJ, I,
        3 * I, 3 * I, CUBLASLT_EPILOGUE_BGRADA, CUDA_R_32F, true);
  probe(h, "bwd' C[I,3I]=X^T dQKV, BGRADB fp32 out", CUDA_R_32F, true, false, I, 3 * I, BJ, I,
        3 * I, 3 * I, CUBLASLT_EPILOGUE_BGRADB, CUDA_R_32F, true);
  return 0;
}
