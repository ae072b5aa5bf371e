// Host-side launchers of the fused sm_100a kernels (internal to libencoder.so).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.cuh"

namespace enc {
// AdamW model-copy segment: flat elements [begin, begin + n) are also written to `out`
// (dtype 0 = bf16, 1 = fp32); begin and n multiples of 4 (mirrors enc_opt_segment)
struct OptSeg {
  int64_t begin;
  int64_t n;
  void* out;
  int dtype;
  int no_decay;
};
constexpr int kOptMaxSegs = 32;
cudaError_t launch_adamw(int64_t n, float* master, float* m1, float* m2, const float* g,
                         const OptSeg* segs, int nseg, double lr, double b1, double b2,
                         double eps, double wd, int step, double gscale, cudaStream_t st);
}  // namespace enc

// Chunks-per-lane dispatch for the warp-per-row operators: a row of n elements has
// nc = n/8 chunks, lane l owns chunks l, l+32, ...; CPL = ceil(nc/32) rounded up to a
// compiled variant (rows up to 4096 elements).
#define ENC_CPL_DISPATCH(nc, ...)                         \
  do {                                                     \
    const int _cpl = ((nc) + 31) / 32;                     \
    if (_cpl <= 1) { constexpr int CPL = 1; __VA_ARGS__; }        \
    else if (_cpl <= 2) { constexpr int CPL = 2; __VA_ARGS__; }   \
    else if (_cpl <= 4) { constexpr int CPL = 4; __VA_ARGS__; }   \
    else if (_cpl <= 8) { constexpr int CPL = 8; __VA_ARGS__; }   \
    else { constexpr int CPL = 16; __VA_ARGS__; }                 \
  } while (0)

// Same, capped at 8 chunks per lane (rows up to 2048 elements); larger rows return
// cudaErrorInvalidValue (the C ABI rejects them first with ENC_EUNSUPPORTED).
#define ENC_CPL_DISPATCH8(nc, ...)                         \
  do {                                                     \
    const int _cpl = ((nc) + 31) / 32;                     \
    if (_cpl <= 1) { constexpr int CPL = 1; __VA_ARGS__; }        \
    else if (_cpl <= 2) { constexpr int CPL = 2; __VA_ARGS__; }   \
    else if (_cpl <= 4) { constexpr int CPL = 4; __VA_ARGS__; }   \
    else if (_cpl <= 8) { constexpr int CPL = 8; __VA_ARGS__; }   \
    else return cudaErrorInvalidValue;                     \
  } while (0)

namespace enc {

// Deterministic column-reduction workspace (owned by enc_ctx).
// A pending fixed-order column-sum finalize: out_q[j] = sum_{r < R} partials[r*ncols +
// q*nper + j].
struct ColsumJob {
  const float* partials = nullptr;
  int R = 0, ncols = 0, nper = 0;
  float *out0 = nullptr, *out1 = nullptr, *out2 = nullptr;
};

struct ReduceWs {
  float* partials;       // device, capacity `cap_floats`
  size_t cap_floats;
  int num_sms;
  ColsumJob* defer = nullptr;   // non-null: record the finalize here instead of launching it
};
// The tail of every column-reducing launcher: finalize now, or record it in ws.defer so the
// caller can batch several finalizes into one launch (launch_colsum_finalize_jobs).
cudaError_t colsum_finish(const ReduceWs& ws, int R, int ncols, int nper, float* out0,
                          float* out1, float* out2, cudaStream_t st);
// One launch finishing up to 4 recorded jobs (their partial regions must not overlap).
cudaError_t launch_colsum_finalize_jobs(const ColsumJob* jobs, int n, cudaStream_t st);

PhiloxKey make_philox_key(float p, uint64_t seed, uint64_t subseq);

// Programmatic dependent launch (ENC_OPT_PDL): launch_k launches `kern` with the
// programmatic-serialization attribute when pdl_enabled(cls) (kernels that call pdl_wait()
// before reading what their stream predecessor wrote), else as a plain launch.  cls: the
// kernel class bit (PDL_* below) of the ENC_OPT_PDL mask.
enum { PDL_LN = 1, PDL_ATTN_FUSED = 2, PDL_ATTN_BH = 4, PDL_WGEMM = 8, PDL_FINAL = 16 };
bool pdl_enabled(int cls);
void pdl_set(int mask);
template <typename Kern, typename... Args>
cudaError_t launch_k(int cls, Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled(cls) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}

// dtype: 0 = bf16, 1 = fp32 (enc_dtype).  All return cudaSuccess or the launch error;
// shape support is checked by the caller (api.cu) through *_supported().
bool rowop_supported(int n_per_row);  // BSB (K), BDRLN (I): chunks-per-lane variants
bool bdrln_bwd_supported(int I, int dtype);  // shared-memory ring fits

cudaError_t launch_dropout_mask(int64_t n, int64_t index0, const PhiloxKey& pk, uint8_t* keep,
                                cudaStream_t st);

cudaError_t launch_aib_fwd(int dtype, int B, int J, int H, int P, const void* qkv,
                           const float* bqkv, void* q, void* k, void* v, cudaStream_t st);
cudaError_t launch_aib_bwd(int dtype, int B, int J, int H, int P, const void* dq,
                           const void* dk, const void* dv, void* dqkv, float* dbqkv,
                           const ReduceWs& ws, cudaStream_t st);

// X[r, :] += bias (in place, [rows, cols], cols % 8 == 0) and deterministic column sums
// out[c] = sum_r X[r, c]: the AIB bias / bias gradient when the QKV contraction output is
// consumed in place (ops_attn.cu).
cudaError_t launch_bias_rows(int dtype, int64_t rows, int cols, void* X, const float* bias,
                             cudaStream_t st);
cudaError_t launch_colsum(int dtype, int rows, int cols, const void* X, float* out,
                          const ReduceWs& ws, cudaStream_t st);
cudaError_t launch_f32_to_bf16(int n, const float* src, void* dst, cudaStream_t st);

// causal: scores of keys k > query j are -inf (J == K)
cudaError_t launch_bsb_fwd(int dtype, int B, int H, int J, int K, float scale, const void* S,
                           const float* mask_bias, const PhiloxKey& pk, int64_t batch_offset,
                           void* P, void* A, cudaStream_t st, int causal = 0);
cudaError_t launch_bsb_bwd(int dtype, int B, int H, int J, int K, float scale, const void* dA,
                           const void* P, const PhiloxKey& pk, int64_t batch_offset, void* dS,
                           cudaStream_t st);

cudaError_t launch_bdrln_fwd(int dtype, int B, int J, int I, const void* Y, const float* bias,
                             const void* R, const float* gamma, const float* beta, float eps,
                             const PhiloxKey& pk, int64_t batch_offset, void* out, void* xhat,
                             float* rstd, cudaStream_t st, int variant = 0,
                             uint8_t* kb_out = nullptr, const uint8_t* kb_in = nullptr);
// variant: 0 = the default kernel for I, 1 = warp-per-row, 2 / 3 / 4 = row-group kernels with
// that many warps per row (when it divides the row; else the default).
// kb_out / kb_in (optional, [B*J][I/8] bytes, R27): the forward stores the keep
// byte of every 8-element chunk it used; a backward (or forward) given them reads them
// instead of evaluating Philox -- same mask, same results.
cudaError_t launch_bdrln_bwd(int dtype, int B, int J, int I, const void* dOut, const void* xhat,
                             const float* rstd, const float* gamma, const PhiloxKey& pk,
                             int64_t batch_offset, void* dz, void* dYpre, float* dgamma,
                             float* dbeta, float* dbias, const ReduceWs& ws, cudaStream_t st,
                             int variant = 0, const uint8_t* kb_in = nullptr);

// Row-group BDRLN variants (ops_ln_rg.cu): 4 warps per row, persistent, TMA row ring.
bool bdrln_rg_supported(int I);
cudaError_t launch_bdrln_fwd_rg(int dtype, int B, int J, int I, const void* Y, const float* bias,
                                const void* R, const float* gamma, const float* beta, float eps,
                                const PhiloxKey& pk, int64_t batch_offset, void* out, void* xhat,
                                float* rstd, cudaStream_t st, int gw = 0,
                                uint8_t* kb_out = nullptr, const uint8_t* kb_in = nullptr);
cudaError_t launch_bdrln_bwd_rg(int dtype, int B, int J, int I, const void* dOut,
                                const void* xhat, const float* rstd, const float* gamma,
                                const PhiloxKey& pk, int64_t batch_offset, void* dz,
                                void* dYpre, float* dgamma, float* dbeta, float* dbias,
                                const ReduceWs& ws, cudaStream_t st, int gw = 0,
                                const uint8_t* kb_in = nullptr);

// keep bytes of a whole dropout site (R27 layout) from Philox chunk g0 (nchunks % 4 == 0)
cudaError_t launch_keep_bytes(int64_t nchunks, int64_t g0, const PhiloxKey& pk, uint8_t* out,
                              cudaStream_t st, int max_ctas = 0);
int balanced_grid(int tiles);   // persistent CTAs for `tiles` in the fewest waves (attn_fused.cu)
cudaError_t launch_bad_fwd(int dtype, int B, int J, int U, const void* Y1, const float* b1,
                           int act, const PhiloxKey& pk, int64_t batch_offset, void* h,
                           void* A1, cudaStream_t st);
// launch_bad_fwd: h may be null (not stored).  launch_bad_bwd: h is the activation input,
// or with b1 non-null the pre-bias contraction output Y1 (h = Y1 + b1 recomputed).
cudaError_t launch_bad_bwd(int dtype, int B, int J, int U, const void* dA1, const void* h,
                           const float* b1,
                           int act, const PhiloxKey& pk, int64_t batch_offset, void* dh,
                           float* db1, const ReduceWs& ws, cudaStream_t st);

cudaError_t launch_bei(int dtype, int64_t n, const void* a, const void* b, void* out,
                       cudaStream_t st);

// Deterministic finalize: out_q[j] = sum_{r < R} partials[r*ncols + q*nper + j] in
// ascending r order (fixed tree), q = 0..nq-1 with nq*nper = ncols.
cudaError_t launch_colsum_finalize(const float* partials, int R, int ncols, int nper,
                                   float* out0, float* out1, float* out2, cudaStream_t st);

// Hand-written tcgen05 attention contractions (attn_gemm.cu), bf16 in / fp32 accumulate /
// bf16 out.  which: 0 S=Q K^T, 1 C=A V (C in [B,J,H,P]), 2 dA=dC V^T (dC in [B,J,H,P]),
// 3 dV=A^T dC, 4 dQ=dS K, 5 dK=dS^T Q; [J x K] operands [B,H,J,K]; P-wide operands with
// row strides ldx / ldy / ldz (map_pop below; ignored for [J x K] operands).
bool attn_gemm_supported(int J, int P);
cudaError_t launch_attn_gemm(int which, int B, int H, int J, int P, const void* X, int64_t ldx,
                             const void* Y, int64_t ldy, void* Z, int64_t ldz, cudaStream_t st,
                             int K = 0);   // K keys (0: K = J)

// Hand-written tcgen05 weight contractions with fused epilogues (wgemm.cu).  Row-major
// C[M,N] = A B: A K-major [M][K] (a_mn = 0) or MN-major [K][M] (a_mn = 1); B K-major [N][K]
// (b_mn = 0) or MN-major [K][N] (b_mn = 1); bf16 operands, fp32 accumulation.
enum { EPI_STORE = 0, EPI_BAD_FWD = 1, EPI_BAD_BWD = 2 };
struct WgemmArgs {
  int M = 0, N = 0, K = 0;
  const void* A = nullptr; int64_t lda = 0; int a_mn = 0;
  const void* B = nullptr; int64_t ldb = 0; int b_mn = 0;
  void* C = nullptr; int64_t ldc = 0; int out_f32 = 0;   // EPI_BAD_FWD: C = h
  int epi = EPI_STORE;
  int beta = 0;                  // EPI_STORE, bf16: C = acc (+ bias) + C
  const float* bias = nullptr;   // [N] fp32 (EPI_STORE optional; EPI_BAD_FWD: b1)
  void* C2 = nullptr; int64_t ldc2 = 0;          // EPI_BAD_FWD: A1
  const void* aux = nullptr; int64_t ldaux = 0;  // EPI_BAD_BWD: h [M][N]
  float* partials = nullptr;     // EPI_BAD_BWD: [ceil(M/128)*4][N] column partials of dh
  int act = 0;
  PhiloxKey pk{};
  int64_t g0 = 0;                // Philox chunk index of element (0, 0)
  // keep bytes ([M][N/8], R27): EPI_BAD_FWD stores them (kb_out), EPI_BAD_BWD --
  // and EPI_BAD_FWD when they were drawn ahead (R29) -- reads them instead of evaluating
  // Philox (kb_in)
  uint8_t* kb_out = nullptr;
  const uint8_t* kb_in = nullptr;
  void* ws = nullptr; size_t ws_bytes = 0;   // split-K slabs (fp32 EPI_STORE outputs)
  int cg = 0;                    // 0 = CTA pairs (cta_group::2) where M > 128, 1 = single CTAs
};
bool wgemm_supported(const WgemmArgs& g);
cudaError_t launch_wgemm(const WgemmArgs& g, int num_sms, cudaStream_t st);
int wgemm_launches(const WgemmArgs& g, int num_sms);   // kernels launch_wgemm launches
int wgemm_partial_rows(const WgemmArgs& g);            // EPI_BAD_BWD partial rows written

// cuTensorMapEncodeTiled resolved at run time (tmap.cu): the library does not link libcuda.
CUresult tmap_encode_tiled(CUtensorMap* map, CUtensorMapDataType dtype, cuuint32_t rank,
                           void* addr, const cuuint64_t* dims, const cuuint64_t* strides,
                           const cuuint32_t* box, const cuuint32_t* estrides,
                           CUtensorMapInterleave il, CUtensorMapSwizzle sw,
                           CUtensorMapL2promotion l2, CUtensorMapFloatOOBfill oob);

// P-wide attention operands (Q, K, V, C and their gradients) are described by a row
// stride `ld` in elements: ld == P is the head-major [B][H][rows][P] layout; any other ld
// is token-major, element (b, h, j, p) at b*rows*ld + j*ld + h*P + p (C / dC: ld = H*P;
// Q/K/V inside the QKV GEMM output [B, J, 3, H, P]: ld = 3*H*P).
// map_pop: bf16 TMA map with coordinates (p, h, row, b), box {64, 1, box_rows, 1}, SW128.
bool map_pop(CUtensorMap* m, const void* ptr, int B, int H, int rows, int P, int64_t ld,
             int box_rows);

// Per-(b, h) tcgen05 contractions over the [J x K] probability / gradient matrices
// (attn_bh.cu): one CTA streams a whole (b, h) matrix once, outputs resident in TMEM.
// bf16, P == 64, J = K a multiple of 128 up to 512.
bool attn_bh_supported(int J, int P);
// dQ / dK may be null (that output is skipped).  ps_* (optional): per-(b, TMEM quarter)
// column sums of the bf16-rounded output, written at ps[(b*4 + q)*ps_ld + h*P + c] (AIB-bwd's
// bias gradient, finished by launch_colsum_finalize over the B*4 partial rows).
// keep (optional): dropout on load -- A is the stored P and the dropout is applied from the
// ENC_KEEP_BITS words while the block is in shared memory; the result is scaled by `scale`.
// gen_pk (R28): the keep words are generated from that Philox site (chunk index with
// batch_offset, R5) by the dropout-on-load warps and written to `keep`, instead of
// read from it
cudaError_t launch_attn_av_bh(int B, int H, int J, int P, const void* A, const void* V,
                              int64_t ldv, void* C, int64_t ldc, const uint32_t* keep,
                              float scale, cudaStream_t st, void* C_lo = nullptr,
                              const PhiloxKey* gen_pk = nullptr, int64_t batch_offset = 0);
cudaError_t launch_attn_dv_bh(int B, int H, int J, int P, const void* A, const void* dC,
                              int64_t lddc, void* dV, int64_t lddv, float* ps_dv, int ps_ld,
                              const uint32_t* keep, float scale, cudaStream_t st);
cudaError_t launch_attn_dqdk_bh(int B, int H, int J, int P, const void* dS, const void* Kt,
                                int64_t ldk, const void* Q, int64_t ldq, void* dQ, int64_t lddq,
                                void* dK, int64_t lddk, float* ps_dq, float* ps_dk, int ps_ld,
                                cudaStream_t st);

// Fused tcgen05 score kernels (attn_fused.cu): QK^T + BSB (writes P, A) and dC V^T +
// BSB-bwd (writes dS), bf16, P == 64, J == 512 (one 128-row tile per CTA round) or J == 128
// (attn_short.cu: whole (b, h) pairs pipelined through TMEM slots; dispatched by the two
// launchers below).
bool attn_fused_supported(int J, int P);
bool attn_short_supported(int J, int P);
cudaError_t launch_attn_qk_bsb_short(int B, int H, int J, int P, float scale, const void* Q,
                                     int64_t ldq, const void* Kt, int64_t ldk,
                                     const float* mask_bias, const PhiloxKey& pk,
                                     int64_t batch_offset, void* Pout, void* Aout,
                                     uint32_t* keep_bits, cudaStream_t st, int causal,
                                     int keep_pre);
cudaError_t launch_attn_da_bsbb_short(int B, int H, int J, int P, float scale, const void* dC,
                                      int64_t lddc, const void* V, int64_t ldv, const void* Pin,
                                      const PhiloxKey& pk, int64_t batch_offset,
                                      const uint32_t* keep_bits, void* dS, cudaStream_t st,
                                      bool high_prio);
// keep_bits: [B,H,J,K/32] keep-flag words (layout in include/encoder.h), written by the
// forward when non-null and read by the backward instead of recomputing Philox when non-null.
// Q, K (fwd) and dC, V (bwd) are P-wide operands with row strides ldq, ldk, lddc, ldv.
cudaError_t launch_attn_qk_bsb(int B, int H, int J, int P, float scale, const void* Q,
                               int64_t ldq, const void* Kt, int64_t ldk, const float* mask_bias,
                               const PhiloxKey& pk, int64_t batch_offset, void* Pout, void* Aout,
                               uint32_t* keep_bits, cudaStream_t st, int causal = 0,
                               int keep_pre = 0, bool high_prio = false);
// keep words of the attention dropout (ENC_KEEP_BITS layout) for [B,H,J,K], K % 64 == 0; the
// fused forward reads them with keep_pre = 1
cudaError_t launch_attn_keep_bits(int B, int H, int J, int K, const PhiloxKey& pk,
                                  int64_t batch_offset, uint32_t* keep_bits, cudaStream_t st);
// QK^T + BSB + A.V in one tcgen05 kernel (R30): P, keep words, C and C's low word
bool attn_fused_av_supported(int J, int P);
cudaError_t launch_attn_qk_bsb_av(int B, int H, int J, int P, float scale, const void* Q,
                                  int64_t ldq, const void* Kt, int64_t ldk, const void* V,
                                  int64_t ldv, const float* mask_bias, const PhiloxKey& pk,
                                  int64_t batch_offset, void* Pout, uint32_t* keep_bits,
                                  void* C, void* C_lo, int64_t ldc, cudaStream_t st,
                                  int causal);
cudaError_t launch_attn_da_bsbb(int B, int H, int J, int P, float scale, const void* dC,
                                int64_t lddc, const void* V, int64_t ldv, const void* Pin,
                                const PhiloxKey& pk, int64_t batch_offset,
                                const uint32_t* keep_bits, void* dS, cudaStream_t st,
                                bool high_prio = false, const void* Chi = nullptr,
                                const void* Clo = nullptr, int64_t ldc = 0);

// Pointer tables for the two-level-strided batched GEMMs of the attention (A.V forward,
// dA/dV backward): the operand [B,J,H,P] with row stride I per (b,h) pair.
cudaError_t launch_make_attn_ptrs(int B, int H, int J, int P, size_t esize, const void* A,
                                  const void* V, const void* C, const void* dA,
                                  const void* dV, void** table, cudaStream_t st);

}  // namespace enc
