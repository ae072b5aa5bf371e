/*
 * encoder.h -- C ABI of the B200-native (sm_100a) data-movement-optimised BERT encoder
 * layer of arXiv 2007.00072 ("Data Movement Is All You Need: A Case Study on Optimizing
 * Transformers").  Library: paper_2007_00072_b200/libencoder.so.
 *
 * Citations: "PAPER.md:n" = /root/reference/PAPER.md line n (the paper's LaTeX source);
 * "DESIGN.md Rn" = reading n of the paper listed in DESIGN.md.
 *
 * Notation (Fig. 1 caption): B batch, J = K sequence length, H heads,
 * P = W key/value projection size, I = H*P embedding size, U FFN width.
 *
 * Conventions for every entry point
 *   - All tensor pointers are DEVICE pointers unless the name ends in _host.
 *   - All calls are asynchronous on `stream` (a cudaStream_t; NULL = legacy default
 *     stream).  No call synchronises the device; results are valid once `stream` has
 *     reached the call.
 *   - Activations and the four weight matrices are in the call's `enc_dtype` (bf16 or
 *     fp32); biases, gamma, beta, LayerNorm statistics and every parameter gradient are
 *     fp32.  bf16 stores round to nearest even; arithmetic is fp32.
 *   - Layouts are row-major with the last dimension contiguous.
 *   - Every data buffer is owned and allocated by the caller; the library only reads
 *     inputs and writes outputs.  Parameter gradients are WRITTEN (not accumulated) and
 *     are SUMS over the local batch (R11).
 *   - Errors: 0 on success, a negative ENC_E* code otherwise.  All argument checks are
 *     made on the host before anything is launched; on error nothing is launched.  No
 *     C++ exception crosses the ABI.  There is no CPU fallback: a missing or failing
 *     device returns ENC_ECUDA.
 *   - Alignment: every tensor pointer must be 16-byte aligned and I, U, K, P must be
 *     multiples of 8 (ENC_EALIGN otherwise).
 *   - Dropout (R5): keep(n) for logical row-major index n (using the GLOBAL
 *     batch index b + batch_offset) is r(n) >= T with T = floor(p*65536 + 1/2) and r(n)
 *     the 16-bit lane (n & 7) of Philox4x32-10(ctr = (n>>3 lo, n>>3 hi, subseq lo,
 *     subseq hi), key = (seed lo, seed hi)); kept values are scaled by 65536/(65536-T).
 *     Masks are never stored: forward and backward regenerate them.  subseq of the
 *     layer's dropout sites = 4*layer_id + site, site 0 attention probabilities, 1
 *     attention output, 2 FFN activation, 3 FFN output.
 *   - An enc_ctx owns a cuBLAS handle, a cuBLAS workspace and a small device workspace
 *     for deterministic column-reduction partials; it may be used by one stream at a
 *     time (calls on different streams must be serialised by the caller).
 */
#ifndef PAPER_2007_00072_ENCODER_H
#define PAPER_2007_00072_ENCODER_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* enc_stream_t; /* == cudaStream_t */

/* ---- error codes ---------------------------------------------------------------- */
#define ENC_OK 0
#define ENC_EINVAL (-1)       /* bad dimension, K != J, W != P, I != H*P, p not in [0,1) */
#define ENC_EALIGN (-2)       /* pointer not 16-byte aligned or I/U/K/P not multiple of 8 */
#define ENC_EDTYPE (-3)       /* unknown enc_dtype */
#define ENC_ECUDA (-4)        /* CUDA launch/runtime error (enc_last_cuda_error) */
#define ENC_ECUBLAS (-5)      /* cuBLAS error */
#define ENC_EUNSUPPORTED (-6) /* shape outside the compiled kernel variants */
#define ENC_ENULL (-7)        /* required pointer is NULL */

typedef enum { ENC_BF16 = 0, ENC_FP32 = 1 } enc_dtype;

/* Activation of the first FFN linear (R6; paper: ReLU). */
typedef enum { ENC_ACT_GELU_ERF = 0, ENC_ACT_GELU_TANH = 1, ENC_ACT_RELU = 2 } enc_act;

/* Dimensions in the paper's notation.  Self-attention: K == J, W == P,
 * I == H*P.  B is the LOCAL batch of this call. */
typedef struct {
  int B, J, K, H, P, W, I, U;
} enc_dims;

/* Layer configuration (R3-R7). */
typedef struct {
  float p_attn;          /* dropout on attention probabilities (site 0) */
  float p_hidden;        /* dropout after out-proj (site 1) and after linear2 (site 3) */
  float p_ffn;           /* dropout after the activation (site 2) */
  uint64_t seed;         /* Philox key */
  uint32_t layer_id;     /* Philox subsequence = 4*layer_id + site */
  int64_t batch_offset;  /* global batch index of local b = 0 (data parallel) */
  float ln_eps;          /* LayerNorm epsilon inside the square root, biased variance */
  int act;               /* enc_act */
} enc_cfg;

/* Parameters, nn.Linear convention y = x W^T (R9).
 * Wqkv [3I,I] (rows: Q heads 0..H-1, then K heads, then V heads, P rows each),
 * Wo [I,I], W1 [U,I], W2 [I,U] in enc_dtype; bqkv [3I], bo [I], b1 [U], b2 [I],
 * g1/be1/g2/be2 [I] (LayerNorm gamma/beta) fp32. */
typedef struct {
  const void *Wqkv, *Wo, *W1, *W2;
  const float *bqkv, *bo, *b1, *b2, *g1, *be1, *g2, *be2;
} enc_params;

/* Parameter gradients, fp32, same shapes as enc_params; written, summed over batch. */
typedef struct {
  float *dWqkv, *dWo, *dW1, *dW2;
  float *dbqkv, *dbo, *db1, *db2, *dg1, *dbe1, *dg2, *dbe2;
} enc_grads;

/* Views into the caller's `saved` buffer (forward -> backward contract).  Q, K, V, P, A in
 * the attention layout [B,H,J,P] / [B,H,J,K]; C, X1, xhat1, xhat2 [B,J,I]; h, A1 [B,J,U]
 * (enc_dtype); rstd1, rstd2 [B,J] fp32.  keep_attn: the attention-dropout keep flags as
 * 1-bit words, [B,H,J,ceil(K/32)] uint32 (ENC_KEEP_BITS layout below), written by the fused
 * forward score kernel and read by the fused backward so it need not regenerate the Philox
 * stream (unused on the other attention paths).  The BDRLN / BAD dropout masks are not
 * stored: their backward regenerates them. */
typedef struct {
  void *Q, *K, *V, *P, *A, *C, *X1, *xhat1, *h, *A1, *xhat2;
  float *rstd1, *rstd2;
  uint32_t* keep_attn;
} enc_saved_view;

/* ENC_KEEP_BITS layout: word w of row (b,h,j) holds the keep flags of columns
 * 32w .. 32w+31; column 32w + 8c + u (c = 0..3, u = 0..7) is bit
 * (u odd ? 31 : 15) - u/2 - 4c.  (u is the 16-bit Philox lane of chunk c: lanes 2i / 2i+1
 * are the low / high halves of output word i, R5; the order falls out of a
 * SIMD-within-a-register compare of the two lanes of a word.) */

/* Views into `scratch` of the backward temporaries, valid after encoder_layer_backward
 * until the next forward/backward call on the same scratch (parity / inspection hook):
 * dY2 (= BDRLN-bwd#2 dYpre), dX1, dYo, dC [B,J,I]; dA1, dh [B,J,U]; dA, dS [B,H,J,K];
 * dQ, dK, dV [B,H,J,P]; dQKV [B,J,3I]. */
typedef struct {
  void *dY2, *dA1, *dh, *dX1, *dYo, *dC, *dA, *dS, *dQ, *dK, *dV, *dQKV;
} enc_bwd_view;

typedef struct enc_ctx enc_ctx;

/* ---- context ---------------------------------------------------------------------- */
/* Creates a context on `device` (cuBLAS handle + 32 MiB cuBLAS workspace + 64 MiB
 * reduction workspace, all device allocations made here and freed by enc_destroy). */
int enc_create(enc_ctx** ctx, int device);
void enc_destroy(enc_ctx* ctx);
const char* enc_strerror(int code);
/* cudaError_t of the last ENC_ECUDA on this thread (0 if none). */
int enc_last_cuda_error(void);
/* Library version string and the SM architecture it was compiled for ("sm_100a"). */
const char* enc_version(void);

/* ---- instrumentation ------------------------------------------------------------- */
/* Operator ids of the layer, in execution order (Table A.1 rows). */
enum {
  ENC_OP_GEMM_QKV = 0, ENC_OP_AIB_FWD, ENC_OP_GEMM_QK, ENC_OP_BSB_FWD, ENC_OP_GEMM_AV,
  ENC_OP_GEMM_OUT, ENC_OP_BDRLN_FWD1, ENC_OP_GEMM_L1, ENC_OP_BAD_FWD, ENC_OP_GEMM_L2,
  ENC_OP_BDRLN_FWD2, ENC_OP_BDRLN_BWD2, ENC_OP_GEMM_L2_DX, ENC_OP_GEMM_L2_DW, ENC_OP_BAD_BWD,
  ENC_OP_GEMM_L1_DX, ENC_OP_GEMM_L1_DW, ENC_OP_BDRLN_BWD1, ENC_OP_GEMM_OUT_DX,
  ENC_OP_GEMM_OUT_DW, ENC_OP_GEMM_AV_DA, ENC_OP_GEMM_AV_DV, ENC_OP_BSB_BWD, ENC_OP_GEMM_QK_DQ,
  ENC_OP_GEMM_QK_DK, ENC_OP_AIB_BWD, ENC_OP_GEMM_QKV_DX, ENC_OP_GEMM_QKV_DW, ENC_NUM_OPS
};
int enc_num_ops(void);
const char* enc_op_name(int op);
/* Record CUDA events on the layer's stream around every operator whose bit (1 << op) is
 * set, in subsequent encoder_layer_forward/backward calls (0 disables). */
int enc_set_timing(enc_ctx* ctx, uint64_t op_mask);
/* ms[op] = device time of the last recorded launch of each timed operator, -1 if not
 * recorded (ms has enc_num_ops() entries).  Waits for those events. */
int enc_op_times(enc_ctx* ctx, float* ms);
/* Number of kernels this library (not cuBLAS) launched through `ctx` so far. */
uint64_t enc_launch_count(const enc_ctx* ctx);

/* ---- whole layer (PAPER.md:129 post-LN BERT layer; Table A.1 order PAPER.md:549-596) */
/* Bytes of the caller-owned `saved` (fwd -> bwd) and `scratch` (temporaries of either
 * pass) buffers for these dims/dtype. */
int enc_layer_sizes(const enc_dims* d, int dtype, size_t* saved_bytes, size_t* scratch_bytes);
/* Pointers to the named tensors inside `saved` (test / inspection hook). */
int enc_saved_views(const enc_dims* d, int dtype, void* saved, enc_saved_view* out);
/* Pointers to the backward temporaries inside `scratch` (test / inspection hook). */
int enc_bwd_views(const enc_dims* d, int dtype, void* scratch, enc_bwd_view* out);

/* Forward: X [B,J,I] -> Y [B,J,I].  mask_bias [B,K] fp32 additive attention bias
 * (BERT key-padding mask, R1) or NULL.  Steps: QKV GEMM, AIB, QK^T, BSB,
 * A.V, Out GEMM, BDRLN#1, Linear1, BAD, Linear2, BDRLN#2. */
int encoder_layer_forward(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                          const enc_params* prm, const void* X, const float* mask_bias,
                          void* Y, void* saved, void* scratch, enc_stream_t stream);
/* Backward: given dY [B,J,I] and the forward's `saved`, writes dX [B,J,I] and all
 * parameter gradients.  X is the forward input (for dWqkv). */
int encoder_layer_backward(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                           const enc_params* prm, const void* X, const void* saved,
                           const void* dY, void* dX, const enc_grads* g, void* scratch,
                           enc_stream_t stream);
/* The backward in two halves, for overlapping the data-parallel gradient all-reduce with
 * the rest of the backward: ENC_BWD_FFN runs BDRLN-bwd#2 .. Linear1 dW (afterwards dW1,
 * dW2, db1, db2, dgamma2, dbeta2 are final), ENC_BWD_ATTN the remainder (BDRLN-bwd#1 ..
 * QKV dW).  Calling both in that order equals encoder_layer_backward. */
enum { ENC_BWD_FFN = 1, ENC_BWD_ATTN = 2 };
int encoder_layer_backward_part(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                                const enc_params* prm, const void* X, const void* saved,
                                const void* dY, void* dX, const enc_grads* g, void* scratch,
                                int part, enc_stream_t stream);
/* End-to-end step from HOST buffers (pinned for overlap): copies X_host, dY_host to
 * X_dev, dY_dev, runs forward + backward, copies Y and dX back to Y_host, dX_host.
 * Parameter gradients stay on the device in `g`. */
int encoder_layer_step_host(enc_ctx* ctx, const enc_dims* d, int dtype, const enc_cfg* cfg,
                            const enc_params* prm, const void* X_host, const void* dY_host,
                            void* Y_host, void* dX_host, void* X_dev, void* dY_dev,
                            void* Y_dev, void* dX_dev, const float* mask_bias,
                            const enc_grads* g, void* saved, void* scratch,
                            enc_stream_t stream);

/* ---- per-operator entry points ----------------------------------------------------- */
/* Dropout keep mask test hook: keep[i] = 1 if logical index index0+i is kept, else 0
 * (uint8, one byte per element, n elements). */
int enc_dropout_mask(int64_t n, int64_t index0, float p, uint64_t seed, uint64_t subseq,
                     uint8_t* keep, enc_stream_t stream);

/* AIB (paper `aib`; Table A.1 :550): q/k/v[B,H,J,P] = permute(qkv[B,J,3I]
 * + bqkv[3I]).  Column block t*I + h*P + p of qkv goes to (t, b, h, j, p). */
int enc_aib_fwd(enc_ctx* ctx, int dtype, int B, int J, int H, int P, const void* qkv,
                const float* bqkv, void* q, void* k, void* v, enc_stream_t stream);
/* AIB-bwd (paper `baib`): dqkv[B,J,3I] = inverse permute of
 * dq/dk/dv [B,H,J,P]; dbqkv[3I] = column sums of dqkv over the B*J rows. */
int enc_aib_bwd(enc_ctx* ctx, int dtype, int B, int J, int H, int P, const void* dq,
                const void* dk, const void* dv, void* dqkv, float* dbqkv,
                enc_stream_t stream);

/* BSB (paper `sm`): P = softmax_k(scale*S + M[b,k]),
 * A = keep*s*P.  S, P, A [B,H,J,K]; mask_bias [B,K] fp32 or NULL; keep indexed on
 * [B,H,J,K] with the global batch index. */
int enc_bsb_fwd(enc_ctx* ctx, int dtype, int B, int H, int J, int K, float scale,
                const void* S, const float* mask_bias, float p, uint64_t seed,
                uint64_t subseq, int64_t batch_offset, void* P, void* A,
                enc_stream_t stream);
/* BSB-bwd (paper `bs`): dP = keep*s*dA,
 * dS = scale * P * (dP - sum_k dP*P). */
int enc_bsb_bwd(enc_ctx* ctx, int dtype, int B, int H, int J, int K, float scale,
                const void* dA, const void* P, float p, uint64_t seed, uint64_t subseq,
                int64_t batch_offset, void* dS, enc_stream_t stream);

/* BDRLN (paper `drln`/`bdrln`):
 * z = R + keep*s*(Y + bias); xhat = (z - mean)/sqrt(var + eps) over I (biased var);
 * out = gamma*xhat + beta.  Y, R, out, xhat [B,J,I]; rstd [B,J] fp32. */
int enc_bdrln_fwd(enc_ctx* ctx, int dtype, int B, int J, int I, const void* Y,
                  const float* bias, const void* R, const float* gamma, const float* beta,
                  float eps, float p, uint64_t seed, uint64_t subseq, int64_t batch_offset,
                  void* out, void* xhat, float* rstd, enc_stream_t stream);
/* BDRLN-bwd (paper `bsb`+`blnrd`+`ebsb`+`baob`):
 * g = dOut*gamma; dz = rstd*(g - mean_I g - xhat*mean_I(g*xhat)); dYpre = keep*s*dz;
 * dgamma = sum_rows dOut*xhat, dbeta = sum_rows dOut, dbias = sum_rows dYpre.
 * dz (the residual gradient) and dYpre [B,J,I]; column sums are deterministic. */
int enc_bdrln_bwd(enc_ctx* ctx, int dtype, int B, int J, int I, const void* dOut,
                  const void* xhat, const float* rstd, const float* gamma, float p,
                  uint64_t seed, uint64_t subseq, int64_t batch_offset, void* dz,
                  void* dYpre, float* dgamma, float* dbeta, float* dbias,
                  enc_stream_t stream);

/* BAD (paper `brd`): h = Y1 + b1; A1 = keep*s*act(h).
 * Y1, h, A1 [B,J,U]. */
int enc_bad_fwd(enc_ctx* ctx, int dtype, int B, int J, int U, const void* Y1,
                const float* b1, int act, float p, uint64_t seed, uint64_t subseq,
                int64_t batch_offset, void* h, void* A1, enc_stream_t stream);
/* BAD-bwd (paper `bdrb`): dh = keep*s*dA1*act'(h);
 * db1 = sum_rows dh. */
int enc_bad_bwd(enc_ctx* ctx, int dtype, int B, int J, int U, const void* dA1,
                const void* h, int act, float p, uint64_t seed, uint64_t subseq,
                int64_t batch_offset, void* dh, float* db1, enc_stream_t stream);

/* Attention contractions on the hand-written tcgen05/TMEM/TMA kernels (bf16 only;
 * J % 128 == 0, P == 64).  which: ENC_AG_QK  S[B,H,J,K] = Q K^T (Table A.1 :551),
 * ENC_AG_AV C[B,J,H,P] = A V (:553), ENC_AG_DA dA = dC V^T (:588, dC in [B,J,H,P]),
 * ENC_AG_DV dV = A^T dC (:589), ENC_AG_DQ dQ = dS K (:591), ENC_AG_DK dK = dS^T Q (:592);
 * Q, K, V, dQ, dK, dV [B,H,J,P]; S, A, dA, dS [B,H,J,K].  X, Y = the two operands in the
 * order written, Z = the result.  With ENC_OPT_ATTN_BH on (default) and J = K a multiple
 * of 128 up to 512, AV / DV / DQ / DK run on the per-(b, h) streaming kernel (one CTA reads a
 * whole [J x K] matrix once, outputs resident in TMEM); otherwise on the tiled kernel. */
enum { ENC_AG_QK = 0, ENC_AG_AV, ENC_AG_DA, ENC_AG_DV, ENC_AG_DQ, ENC_AG_DK };
int enc_attn_gemm(enc_ctx* ctx, int which, int B, int H, int J, int P, const void* X,
                  const void* Y, void* Z, enc_stream_t stream);

/* Fused score kernels (bf16, P == 64, J == K == 512, the paper's sequence length): one
 * tcgen05 kernel computes the contraction into TMEM and applies the fused normalisation in
 * its epilogue, so the score tensor never reaches HBM.
 *   enc_attn_fwd_fused: S = Q K^T (:551) then BSB (:552) -> P, A [B,H,J,K]
 *   enc_attn_bwd_fused: dA = dC V^T (:588, dC in [B,J,H,P]) then BSB-bwd (:590) with the
 *                       saved P -> dS [B,H,J,K]
 * Same dropout / scale conventions as enc_bsb_fwd / enc_bsb_bwd.  keep_bits (optional,
 * 8-B aligned, [B,H,J,K/32] uint32, ENC_KEEP_BITS layout): the forward writes the keep
 * flags it used there; the backward, given the forward's words, reads them instead of
 * regenerating the Philox stream (null: regenerate; both give the same dS). */
int enc_attn_fwd_fused(enc_ctx* ctx, int B, int H, int J, int P, float scale, const void* Q,
                       const void* K, const float* mask_bias, float p, uint64_t seed,
                       uint64_t subseq, int64_t batch_offset, void* P_out, void* A,
                       uint32_t* keep_bits, enc_stream_t stream);
int enc_attn_bwd_fused(enc_ctx* ctx, int B, int H, int J, int P, float scale, const void* dC,
                       const void* V, const void* P_in, float p, uint64_t seed, uint64_t subseq,
                       int64_t batch_offset, const uint32_t* keep_bits, void* dS,
                       enc_stream_t stream);

/* Options of a context.  ENC_OPT_ATTN_TC: 1 = the layer runs its attention contractions on
 * the hand-written tcgen05 kernels (default when supported), 0 = cuBLAS.
 * ENC_OPT_ATTN_FUSED: 1 = QK^T+BSB and dA+BSB-bwd run as the fused kernels above (default
 * when supported; requires ENC_OPT_ATTN_TC), 0 = separate contraction and BSB kernels. */
/* ENC_OPT_GEMM_LT: 1 = the weight contractions (QKV, Out, Linear1/2, fwd/dX/dW) run through
 * cuBLASLt with a per-shape algorithm chosen by timing every heuristic candidate on the
 * first eager call (the paper's contraction tuning; default), 0 = cuBLAS
 * cublasGemmEx with its default heuristic.  ENC_OPT_GEMM_AUTOTUNE: 1 = measure (default),
 * 0 = take cuBLASLt's first heuristic candidate.  ENC_OPT_ATTN_BH: 1 = the AV / dV / dQ+dK
 * contractions run on the per-(b, h) streaming kernel when supported (default; the layer
 * then computes dQ and dK in one pass over dS), 0 = the tiled tcgen05 kernel. */
enum { ENC_OPT_ATTN_TC = 0, ENC_OPT_ATTN_FUSED = 1, ENC_OPT_GEMM_LT = 2, ENC_OPT_GEMM_AUTOTUNE = 3,
       ENC_OPT_ATTN_BH = 4 };
int enc_set_option(enc_ctx* ctx, int key, int value);

/* BEI (paper `bei`): out = a + b, n elements (out may alias a). */
int enc_bei(enc_ctx* ctx, int dtype, int64_t n, const void* a, const void* b, void* out,
            enc_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
