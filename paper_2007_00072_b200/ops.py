"""Per-operator Python binding: the same names as include/encoder.h, taking torch CUDA
tensors.  Argument marshalling only (pointers, sizes, the current CUDA stream); every
step runs in libencoder.so.  PyTorch supplies device memory and streams only."""
from __future__ import annotations

import torch

from . import _abi
from ._abi import check

_DT = {torch.bfloat16: _abi.ENC_BF16, torch.float32: _abi.ENC_FP32}


def _dt(t: torch.Tensor) -> int:
    if t.dtype not in _DT:
        raise TypeError(f"unsupported dtype {t.dtype}")
    return _DT[t.dtype]


def _p(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("tensor must be on a CUDA device (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Context:
    """Owns an enc_ctx (cuBLAS handle, cuBLAS workspace, reduction workspace)."""

    def __init__(self, device=None):
        lib = _abi.load()
        dev = torch.cuda.current_device() if device is None else int(device)
        h = _abi.c_void_p()
        check("enc_create", lib.enc_create(_abi.ctypes.byref(h), dev))
        self.handle = h
        self.device = dev
        self._lib = lib

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.enc_destroy(h)
            self.handle = None

    @property
    def ptr(self):
        return self.handle


def enc_dropout_mask(n, index0, p, seed, subseq, keep: torch.Tensor, stream=None):
    lib = _abi.load()
    check("enc_dropout_mask", lib.enc_dropout_mask(n, index0, p, seed, subseq, _p(keep),
                                                   _stream(stream)))


def enc_aib_fwd(ctx, B, J, H, P, qkv, bqkv, q, k, v, stream=None):
    check("enc_aib_fwd", _abi.load().enc_aib_fwd(ctx.ptr, _dt(qkv), B, J, H, P, _p(qkv), _p(bqkv),
                                                 _p(q), _p(k), _p(v), _stream(stream)))


def enc_aib_bwd(ctx, B, J, H, P, dq, dk, dv, dqkv, dbqkv, stream=None):
    check("enc_aib_bwd", _abi.load().enc_aib_bwd(ctx.ptr, _dt(dq), B, J, H, P, _p(dq), _p(dk),
                                                 _p(dv), _p(dqkv), _p(dbqkv), _stream(stream)))


def enc_bsb_fwd(ctx, B, H, J, K, scale, S, mask_bias, p, seed, subseq, batch_offset, P, A,
                stream=None, causal=False):
    check("enc_bsb_fwd", _abi.load().enc_bsb_fwd(ctx.ptr, _dt(S), B, H, J, K, scale, _p(S),
                                                 _p(mask_bias), p, seed, subseq, batch_offset,
                                                 _p(P), _p(A), int(causal), _stream(stream)))


def enc_bsb_bwd(ctx, B, H, J, K, scale, dA, P, p, seed, subseq, batch_offset, dS, stream=None):
    check("enc_bsb_bwd", _abi.load().enc_bsb_bwd(ctx.ptr, _dt(dA), B, H, J, K, scale, _p(dA),
                                                 _p(P), p, seed, subseq, batch_offset, _p(dS),
                                                 _stream(stream)))


def enc_bdrln_fwd(ctx, B, J, I, Y, bias, R, gamma, beta, eps, p, seed, subseq, batch_offset,
                  out, xhat, rstd, stream=None):
    check("enc_bdrln_fwd", _abi.load().enc_bdrln_fwd(
        ctx.ptr, _dt(Y), B, J, I, _p(Y), _p(bias), _p(R), _p(gamma), _p(beta), eps, p, seed,
        subseq, batch_offset, _p(out), _p(xhat), _p(rstd), _stream(stream)))


def enc_bdrln_bwd(ctx, B, J, I, dOut, xhat, rstd, gamma, p, seed, subseq, batch_offset, dz,
                  dYpre, dgamma, dbeta, dbias, stream=None):
    check("enc_bdrln_bwd", _abi.load().enc_bdrln_bwd(
        ctx.ptr, _dt(dOut), B, J, I, _p(dOut), _p(xhat), _p(rstd), _p(gamma), p, seed, subseq,
        batch_offset, _p(dz), _p(dYpre), _p(dgamma), _p(dbeta), _p(dbias), _stream(stream)))


def enc_bad_fwd(ctx, B, J, U, Y1, b1, act, p, seed, subseq, batch_offset, h, A1, stream=None):
    check("enc_bad_fwd", _abi.load().enc_bad_fwd(ctx.ptr, _dt(Y1), B, J, U, _p(Y1), _p(b1), act,
                                                 p, seed, subseq, batch_offset, _p(h), _p(A1),
                                                 _stream(stream)))


def enc_bad_bwd(ctx, B, J, U, dA1, h, act, p, seed, subseq, batch_offset, dh, db1, stream=None):
    check("enc_bad_bwd", _abi.load().enc_bad_bwd(ctx.ptr, _dt(dA1), B, J, U, _p(dA1), _p(h), act,
                                                 p, seed, subseq, batch_offset, _p(dh), _p(db1),
                                                 _stream(stream)))


def enc_bei(ctx, a, b, out, stream=None):
    check("enc_bei", _abi.load().enc_bei(ctx.ptr, _dt(a), a.numel(), _p(a), _p(b), _p(out),
                                         _stream(stream)))


AG_QK, AG_AV, AG_DA, AG_DV, AG_DQ, AG_DK = range(6)


def enc_attn_gemm(ctx, which, B, H, J, P, X, Y, Z, stream=None):
    check("enc_attn_gemm", _abi.load().enc_attn_gemm(ctx.ptr, which, B, H, J, P, _p(X), _p(Y),
                                                     _p(Z), _stream(stream)))


def enc_set_option(ctx, key, value):
    check("enc_set_option", _abi.load().enc_set_option(ctx.ptr, key, value))


(OPT_ATTN_TC, OPT_ATTN_FUSED, OPT_GEMM_LT, OPT_GEMM_AUTOTUNE, OPT_ATTN_BH, OPT_QKV_DIRECT,
 OPT_BWD_SIDE, OPT_ATTN_OVERLAP, OPT_GEMM_TC, OPT_GEMM_PAIR, OPT_GEMM_TC_MASK,
 OPT_KEEP_AHEAD, OPT_QKV_FUSION, OPT_QKV_FUSION_BWD, OPT_BDRLN_VARIANT, OPT_ATTN_DC,
 OPT_MASK_BYTES, OPT_PDL, OPT_AV_KEEP_GEN, OPT_MASK_AHEAD, OPT_SIDE_OPS,
 OPT_ATTN_FUSED_AV) = range(22)
QKV_SEPARATE, QKV_QK_STACKED, QKV_STACKED, QKV_KV_STACKED = range(4)


def enc_attn_fwd_fused(ctx, B, H, J, P, scale, Q, K, mask_bias, p, seed, subseq, batch_offset,
                       Pout, A, keep_bits=None, stream=None, causal=False):
    check("enc_attn_fwd_fused", _abi.load().enc_attn_fwd_fused(
        ctx.ptr, B, H, J, P, scale, _p(Q), _p(K), _p(mask_bias), p, seed, subseq, batch_offset,
        _p(Pout), _p(A), _p(keep_bits), int(causal), _stream(stream)))


def enc_attn_bwd_fused(ctx, B, H, J, P, scale, dC, V, Pin, p, seed, subseq, batch_offset, dS,
                       keep_bits=None, stream=None):
    check("enc_attn_bwd_fused", _abi.load().enc_attn_bwd_fused(
        ctx.ptr, B, H, J, P, scale, _p(dC), _p(V), _p(Pin), p, seed, subseq, batch_offset,
        _p(keep_bits), _p(dS), _stream(stream)))


def enc_attn_fwd_fused_av(ctx, B, H, J, P, scale, Q, K, V, mask_bias, p, seed, subseq,
                          batch_offset, Pout, keep_bits, C, C_lo, stream=None, causal=False):
    check("enc_attn_fwd_fused_av", _abi.load().enc_attn_fwd_fused_av(
        ctx.ptr, B, H, J, P, scale, _p(Q), _p(K), _p(V), _p(mask_bias), p, seed, subseq,
        batch_offset, _p(Pout), _p(keep_bits), _p(C), _p(C_lo), int(causal), _stream(stream)))


def enc_attn_bwd_fused_dc(ctx, B, H, J, P, scale, dC, V, Pin, C_hi, C_lo, p, seed, subseq,
                          batch_offset, dS, keep_bits=None, stream=None):
    check("enc_attn_bwd_fused_dc", _abi.load().enc_attn_bwd_fused_dc(
        ctx.ptr, B, H, J, P, scale, _p(dC), _p(V), _p(Pin), _p(C_hi), _p(C_lo), p, seed,
        subseq, batch_offset, _p(keep_bits), _p(dS), _stream(stream)))


def enc_wgemm(ctx, A, B, C, tA=False, tB=False, beta=0, bias=None, M=None, N=None, K=None,
              stream=None):
    """C[M,N] = op(A) op(B) (+ bias) (+ C) on the tcgen05 weight-contraction kernel; A, B
    bf16 row-major ([M,K] or, tA, [K,M]; [K,N] or, tB, [N,K]); C bf16 or fp32 [M,N]."""
    if A.dtype != torch.bfloat16 or B.dtype != torch.bfloat16:
        raise TypeError("enc_wgemm takes bf16 operands")
    M = C.shape[0] if M is None else M
    N = C.shape[1] if N is None else N
    K = (A.shape[0] if tA else A.shape[1]) if K is None else K
    check("enc_wgemm", _abi.load().enc_wgemm(
        ctx.ptr, M, N, K, _p(A), A.stride(0), int(tA), _p(B), B.stride(0), int(tB), _p(C),
        C.stride(0), _dt(C), int(beta), _p(bias), _stream(stream)))


def enc_linear1_bad_fwd(ctx, B, J, I, U, X1, W1, b1, act, p, seed, subseq, batch_offset, h, A1,
                        stream=None):
    check("enc_linear1_bad_fwd", _abi.load().enc_linear1_bad_fwd(
        ctx.ptr, B, J, I, U, _p(X1), _p(W1), _p(b1), act, p, seed, subseq, batch_offset, _p(h),
        _p(A1), _stream(stream)))


def enc_linear2_dx_bad_bwd(ctx, B, J, I, U, dY2, W2, h, act, p, seed, subseq, batch_offset, dh,
                           db1, stream=None):
    check("enc_linear2_dx_bad_bwd", _abi.load().enc_linear2_dx_bad_bwd(
        ctx.ptr, B, J, I, U, _p(dY2), _p(W2), _p(h), act, p, seed, subseq, batch_offset, _p(dh),
        _p(db1), _stream(stream)))


def enc_attn_keep_bits(ctx, B, H, J, K, p, seed, subseq, batch_offset, keep_bits, stream=None):
    check("enc_attn_keep_bits", _abi.load().enc_attn_keep_bits(
        ctx.ptr, B, H, J, K, p, seed, subseq, batch_offset, _p(keep_bits), _stream(stream)))


def enc_attn_fwd_fused_bits(ctx, B, H, J, P, scale, Q, K, mask_bias, p, seed, subseq,
                            batch_offset, Pout, A, keep_bits, stream=None, causal=False):
    check("enc_attn_fwd_fused_bits", _abi.load().enc_attn_fwd_fused_bits(
        ctx.ptr, B, H, J, P, scale, _p(Q), _p(K), _p(mask_bias), p, seed, subseq, batch_offset,
        _p(Pout), _p(A), _p(keep_bits), int(causal), _stream(stream)))
