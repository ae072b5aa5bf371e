"""Oracle: plain fp64 BERT encoder layer, forward and backward, per operator.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Slow, obviously-correct numpy in
float64.  Library primitives used as single steps: numpy matmul/einsum (contractions),
scipy.special.erf.  No blocking, fusion or reordering beyond the definitions.

Fusion and layout selection do not change values ("does not change the
underlying computation"), so each fused operator below is the plain composition of the
unfused operators of Table A.1 in that table's order.  Names follow
the north star (BSB, BDRLN, BAD, AIB, BEI); the crosswalk to the paper's kernel names
(sm, drln/bdrln, brd, bs, blnrd/bsb/ebsb/baob, bdrb, aib/baib, bei) is
in DESIGN.md.

Notation: B batch, J = K sequence length, H heads, P = W head size,
I = H*P, U = FFN width.  Tensors are numpy arrays; every input is promoted to float64.
Readings of points the paper leaves open are DESIGN.md R1..R17.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.special import erf

from . import philox

F64 = np.float64

ACT_GELU_ERF = 0
ACT_GELU_TANH = 1
ACT_RELU = 2

SITE_ATTN = 0      # dropout on attention probabilities (paper `sm`)
SITE_ATTN_OUT = 1  # dropout after the output projection (paper `drln`)
SITE_FFN = 2       # dropout after the activation (paper `brd`)
SITE_FFN_OUT = 3   # dropout after linear2 (paper `bdrln`)


@dataclass
class Cfg:
    """Layer configuration (R3, R4, R7)."""
    p_attn: float = 0.1
    p_hidden: float = 0.1
    p_ffn: float = 0.1
    seed: int = 2007000072
    layer_id: int = 0
    batch_offset: int = 0
    ln_eps: float = 1e-5
    act: int = ACT_GELU_ERF
    causal: bool = False   # DESIGN.md R22: key k > query j masked out


def _f(a):
    return None if a is None else np.asarray(a, dtype=F64)


def _mask(shape, p, seed, subseq, batch_offset):
    """(keep mask as float64 0/1, scale s) for a dropout site (oracle/philox.py)."""
    keep = philox.keep_mask_tensor(shape, batch_offset, p, seed, subseq)
    return keep.astype(F64), philox.dropout_scale(p)


# ----------------------------------------------------------------------------------
# Activations (R6).  Paper: ReLU; north star: GELU/ReLU.
# ----------------------------------------------------------------------------------
def act_fwd(h, act):
    h = _f(h)
    if act == ACT_GELU_ERF:
        return 0.5 * h * (1.0 + erf(h / np.sqrt(2.0)))
    if act == ACT_GELU_TANH:
        c = np.sqrt(2.0 / np.pi)
        return 0.5 * h * (1.0 + np.tanh(c * (h + 0.044715 * h ** 3)))
    if act == ACT_RELU:
        return np.maximum(h, 0.0)
    raise ValueError(act)


def act_bwd(h, act):
    """d act(h) / dh."""
    h = _f(h)
    if act == ACT_GELU_ERF:
        return 0.5 * (1.0 + erf(h / np.sqrt(2.0))) + h * np.exp(-0.5 * h * h) / np.sqrt(2.0 * np.pi)
    if act == ACT_GELU_TANH:
        c = np.sqrt(2.0 / np.pi)
        t = np.tanh(c * (h + 0.044715 * h ** 3))
        return 0.5 * (1.0 + t) + 0.5 * h * (1.0 - t * t) * c * (1.0 + 3.0 * 0.044715 * h * h)
    if act == ACT_RELU:
        return (h > 0.0).astype(F64)   # ReLU'(0) = 0
    raise ValueError(act)


# ----------------------------------------------------------------------------------
# AIB: attention input bias (paper `aib`; Table A.1 "Input bias" :550)
# ----------------------------------------------------------------------------------
def aib_fwd(QKV, bqkv, H, P):
    """QKV [B,J,3I] (stacked Q|K|V projections, PAPER.md:640 algebraic QKV fusion) plus
    b_qkv [3I]; returns Q, K, V in the attention layout [B,H,J,P].  Head h of Q uses
    columns [h*P, (h+1)*P) of the first I outputs, K and V the second and third thirds
    (R9)."""
    QKV = _f(QKV) + _f(bqkv)
    B, J, I3 = QKV.shape
    I = I3 // 3
    parts = QKV.reshape(B, J, 3, H, P)
    return tuple(np.ascontiguousarray(parts[:, :, t].transpose(0, 2, 1, 3)) for t in range(3))


def aib_bwd(dQ, dK, dV):
    """Paper `baib` (Table A.1 "Input bias dW" :595): inverse permute of
    dQ, dK, dV [B,H,J,P] into dQKV [B,J,3I] and the bias gradient, a column sum over
    all B*J rows."""
    dQ, dK, dV = _f(dQ), _f(dK), _f(dV)
    B, H, J, P = dQ.shape
    dQKV = np.stack([t.transpose(0, 2, 1, 3) for t in (dQ, dK, dV)], axis=2).reshape(B, J, 3 * H * P)
    return dQKV, dQKV.sum(axis=(0, 1))


# ----------------------------------------------------------------------------------
# BSB: (bias +) scaled softmax + dropout on attention scores (paper `sm`, PAPER.md:514;
# Table A.1 "Scaled softmax" :552).  Backward: paper `bs`.
# ----------------------------------------------------------------------------------
def bsb_fwd(S, mask_bias, scale, p, seed, subseq, batch_offset=0, causal=False):
    """S [B,H,J,K] raw scores Q.K^T; mask_bias [B,K] additive (R1) or None.
    P = softmax_k(scale*S + M[b,k]) (row max subtracted, "multiplied
    together and scaled ... followed by a softmax"); A = P * keep * s.
    causal: the masking step that keeps a query from "seeing the future":
    scores of keys k > j are -inf, so P[..., j, k] = 0 there (R22).
    Returns (P, A)."""
    S = _f(S)
    x = scale * S
    if mask_bias is not None:
        x = x + _f(mask_bias)[:, None, None, :]
    if causal:
        J, K = S.shape[-2], S.shape[-1]
        x = np.where(np.arange(K)[None, :] > np.arange(J)[:, None], -np.inf, x)
    x = x - x.max(axis=-1, keepdims=True)
    e = np.exp(x)
    Pm = e / e.sum(axis=-1, keepdims=True)
    keep, s = _mask(S.shape, p, seed, subseq, batch_offset)
    return Pm, Pm * keep * s


def bsb_bwd(dA, Pm, scale, p, seed, subseq, batch_offset=0):
    """dP = keep*s*dA;  dS = scale * P * (dP - sum_k dP*P)  (softmax Jacobian-vector
    product; the scale is the chain rule through scale*S)."""
    dA, Pm = _f(dA), _f(Pm)
    keep, s = _mask(dA.shape, p, seed, subseq, batch_offset)
    dP = dA * keep * s
    return scale * Pm * (dP - (dP * Pm).sum(axis=-1, keepdims=True))


# ----------------------------------------------------------------------------------
# BDRLN: bias + dropout + residual + LayerNorm (paper `drln`/`bdrln`, PAPER.md:516;
# Table A.1 :555-558 and :564-567).  Backward: paper `bsb` (LN dW, :517/:570),
# `blnrd` (LN dX + dropout dX, :518/:571-572, :583-584), `ebsb` (:520/:581-582),
# `baob` / bias2-dW part of `bdrb` (:512/:585, :575).
# ----------------------------------------------------------------------------------
def bdrln_fwd(Y, bias, R, gamma, beta, eps, p, seed, subseq, batch_offset=0):
    """z = R + keep*s*(Y + bias);  x^ = (z - mu) / sqrt(var + eps) with the BIASED
    mean/variance over the last dim (R7);  out = gamma*x^ + beta.
    Y, R [B,J,I].  Returns (out, xhat, rstd [B,J])."""
    Y, R = _f(Y), _f(R)
    keep, s = _mask(Y.shape, p, seed, subseq, batch_offset)
    z = R + keep * s * (Y + _f(bias))
    mu = z.mean(axis=-1, keepdims=True)
    var = ((z - mu) ** 2).mean(axis=-1, keepdims=True)
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (z - mu) * rstd
    return _f(gamma) * xhat + _f(beta), xhat, rstd[..., 0]


def bdrln_bwd(dOut, xhat, rstd, gamma, p, seed, subseq, batch_offset=0):
    """Given dOut = dL/d(out):
        dgamma = sum_rows dOut*x^,  dbeta = sum_rows dOut              (LN dW)
        g  = dOut*gamma
        dz = rstd * (g - mean_I(g) - x^ * mean_I(g*x^))                (LN dX)
        dYpre = keep*s*dz  (grad w.r.t. Y and the bias; dropout dX)
        dbias = sum_rows dYpre                                         (bias dW)
    dz is also the gradient flowing into the residual input R.
    Returns (dz, dYpre, dgamma, dbeta, dbias)."""
    dOut, xhat = _f(dOut), _f(xhat)
    rstd = _f(rstd)[..., None]
    g = dOut * _f(gamma)
    dz = rstd * (g - g.mean(axis=-1, keepdims=True) - xhat * (g * xhat).mean(axis=-1, keepdims=True))
    keep, s = _mask(dOut.shape, p, seed, subseq, batch_offset)
    dYpre = keep * s * dz
    rows = tuple(range(dOut.ndim - 1))
    return dz, dYpre, (dOut * xhat).sum(axis=rows), dOut.sum(axis=rows), dYpre.sum(axis=rows)


# ----------------------------------------------------------------------------------
# BAD: bias + activation + dropout (paper `brd`).
# Backward: paper `bdrb`.
# ----------------------------------------------------------------------------------
def bad_fwd(Y1, b1, act, p, seed, subseq, batch_offset=0):
    """h = Y1 + b1 (saved);  A1 = keep*s*act(h).  Returns (h, A1)."""
    h = _f(Y1) + _f(b1)
    keep, s = _mask(h.shape, p, seed, subseq, batch_offset)
    return h, keep * s * act_fwd(h, act)


def bad_bwd(dA1, h, act, p, seed, subseq, batch_offset=0):
    """dh = keep*s*dA1 * act'(h);  db1 = sum_rows dh.  Returns (dh, db1)."""
    dA1 = _f(dA1)
    keep, s = _mask(dA1.shape, p, seed, subseq, batch_offset)
    dh = keep * s * dA1 * act_bwd(h, act)
    return dh, dh.sum(axis=tuple(range(dh.ndim - 1)))


def bei(dX_qkv, dz1):
    """Paper `bei`: backward encoder-input residual add."""
    return _f(dX_qkv) + _f(dz1)


# ----------------------------------------------------------------------------------
# Whole layer (post-LN BERT encoder, PAPER.md:129 and Table A.1 operator order)
# ----------------------------------------------------------------------------------
def _lin(x, W):
    """nn.Linear convention y = x W^T (R9)."""
    return np.matmul(x, _f(W).T)


def encoder_layer_forward(X, prm, H, cfg: Cfg, mask_bias=None):
    """Forward pass, Table A.1 forward rows.  Returns (Y, saved)."""
    X = _f(X)
    B, J, I = X.shape
    P = I // H
    scale = 1.0 / np.sqrt(P)                                    # DESIGN.md R3
    sub = lambda site: philox.subsequence(cfg.layer_id, site)   # noqa: E731
    QKV = _lin(X, prm["Wqkv"])                                  # Q,K,V (:549)
    Q, K, V = aib_fwd(QKV, prm["bqkv"], H, P)                   # input bias (:550)
    S = np.matmul(Q, K.transpose(0, 1, 3, 2))                   # QK^T (:551)
    Pm, A = bsb_fwd(S, mask_bias, scale, cfg.p_attn, cfg.seed, sub(SITE_ATTN), cfg.batch_offset,
                    causal=cfg.causal)
    Cbh = np.matmul(A, V)                                       # Gamma (:553), [B,H,J,P]
    C = Cbh.transpose(0, 2, 1, 3).reshape(B, J, I)              # concatenate heads
    Yo = _lin(C, prm["Wo"])                                     # Out (:554)
    X1, xhat1, rstd1 = bdrln_fwd(Yo, prm["bo"], X, prm["g1"], prm["be1"], cfg.ln_eps,
                                 cfg.p_hidden, cfg.seed, sub(SITE_ATTN_OUT), cfg.batch_offset)
    Y1 = _lin(X1, prm["W1"])                                    # Linear (:559)
    h, A1 = bad_fwd(Y1, prm["b1"], cfg.act, cfg.p_ffn, cfg.seed, sub(SITE_FFN), cfg.batch_offset)
    Y2 = _lin(A1, prm["W2"])                                    # Linear (:563)
    Y, xhat2, rstd2 = bdrln_fwd(Y2, prm["b2"], X1, prm["g2"], prm["be2"], cfg.ln_eps,
                                cfg.p_hidden, cfg.seed, sub(SITE_FFN_OUT), cfg.batch_offset)
    saved = dict(QKV=QKV, Q=Q, K=K, V=V, S=S, P=Pm, A=A, C=C, Yo=Yo, X1=X1, xhat1=xhat1,
                 rstd1=rstd1, Y1=Y1, h=h, A1=A1, Y2=Y2, xhat2=xhat2, rstd2=rstd2, Y=Y)
    return Y, saved


def encoder_layer_backward(dY, X, prm, H, cfg: Cfg, saved):
    """Backward pass, Table A.1 backward rows in that order.
    Parameter gradients are SUMS over the local batch (R11).
    Returns (dX, grads, inter)."""
    dY, X = _f(dY), _f(X)
    B, J, I = X.shape
    P = I // H
    scale = 1.0 / np.sqrt(P)
    sub = lambda site: philox.subsequence(cfg.layer_id, site)   # noqa: E731
    sv = saved
    # BDRLN-bwd site 2: LN dW (:570), LN dX + dropout dX (:571-572), bias2 dW (:575)
    dz2, dY2, dg2, dbe2, db2 = bdrln_bwd(dY, sv["xhat2"], sv["rstd2"], prm["g2"],
                                         cfg.p_hidden, cfg.seed, sub(SITE_FFN_OUT), cfg.batch_offset)
    dA1 = np.matmul(dY2, _f(prm["W2"]))                          # Linear dX (:573)
    dW2 = np.einsum("bji,bju->iu", dY2, sv["A1"])                # Linear dW (:574)
    # BAD-bwd: dropout dX, act dX, bias1 dW (:576-578)
    dh, db1 = bad_bwd(dA1, sv["h"], cfg.act, cfg.p_ffn, cfg.seed, sub(SITE_FFN), cfg.batch_offset)
    dX1 = np.matmul(dh, _f(prm["W1"])) + dz2                     # Linear dX (:579) + residual (:581)
    dW1 = np.einsum("bju,bji->ui", dh, sv["X1"])                 # Linear dW (:580)
    # BDRLN-bwd site 1: LN dW (:582), LN dX + dropout dX (:583-584), out bias dW (:585)
    dz1, dYo, dg1, dbe1, dbo = bdrln_bwd(dX1, sv["xhat1"], sv["rstd1"], prm["g1"],
                                         cfg.p_hidden, cfg.seed, sub(SITE_ATTN_OUT), cfg.batch_offset)
    dC = np.matmul(dYo, _f(prm["Wo"]))                           # Out dX (:586)
    dWo = np.einsum("bji,bjk->ik", dYo, sv["C"])                 # Out dW (:587)
    dCbh = dC.reshape(B, J, H, P).transpose(0, 2, 1, 3)
    dA = np.matmul(dCbh, sv["V"].transpose(0, 1, 3, 2))          # Gamma dX1 (:588)
    dV = np.matmul(sv["A"].transpose(0, 1, 3, 2), dCbh)          # Gamma dX2 (:589)
    dS = bsb_bwd(dA, sv["P"], scale, cfg.p_attn, cfg.seed, sub(SITE_ATTN), cfg.batch_offset)
    dQ = np.matmul(dS, sv["K"])                                  # QK^T dX1 (:591)
    dK = np.matmul(dS.transpose(0, 1, 3, 2), sv["Q"])            # QK^T dX2 (:592)
    dQKV, dbqkv = aib_bwd(dQ, dK, dV)                            # input bias dW (:595)
    dXqkv = np.matmul(dQKV, _f(prm["Wqkv"]))                     # Q,K,V dX (:593)
    dWqkv = np.einsum("bjo,bji->oi", dQKV, X)                    # Q,K,V dW (:594)
    dX = bei(dXqkv, dz1)                                         # residual (:596)
    grads = dict(Wqkv=dWqkv, bqkv=dbqkv, Wo=dWo, bo=dbo, W1=dW1, b1=db1, W2=dW2, b2=db2,
                 g1=dg1, be1=dbe1, g2=dg2, be2=dbe2)
    inter = dict(dz2=dz2, dY2=dY2, dA1=dA1, dh=dh, dX1=dX1, dz1=dz1, dYo=dYo, dC=dC, dA=dA,
                 dV=dV, dS=dS, dQ=dQ, dK=dK, dQKV=dQKV)
    return dX, grads, inter


# ----------------------------------------------------------------------------------
# Encoder-decoder (cross) attention sublayer -- the second workload of SURVEY.md 8(f)4:
# queries from the decoder stream X [B,J,I], keys and values from the encoder memory
# Mem [B,K,I] projected by one stacked weight [W^K W^V] (the algebraic "fuse keys and
# values in encoder/decoder attention"), then the same BSB (site 0) and
# BDRLN (site 1, residual X, post-LN) as the encoder layer.  K may differ from J.
# ----------------------------------------------------------------------------------
def cross_attention_forward(X, Mem, prm, H, cfg: Cfg, mask_bias=None):
    """prm: Wq [I,I], Wkv [2I,I], Wo [I,I], bq [I], bkv [2I], bo [I], g, be [I].
    Returns (Y, saved)."""
    X, Mem = _f(X), _f(Mem)
    B, J, I = X.shape
    K = Mem.shape[1]
    P = I // H
    scale = 1.0 / np.sqrt(P)
    sub = lambda site: philox.subsequence(cfg.layer_id, site)   # noqa: E731
    Qf = _lin(X, prm["Wq"]) + _f(prm["bq"])                      # [B,J,I]
    KV = _lin(Mem, prm["Wkv"]) + _f(prm["bkv"])                  # [B,K,2I] keys | values
    Q = Qf.reshape(B, J, H, P).transpose(0, 2, 1, 3)
    Kh = KV[..., :I].reshape(B, K, H, P).transpose(0, 2, 1, 3)
    V = KV[..., I:].reshape(B, K, H, P).transpose(0, 2, 1, 3)
    S = np.matmul(Q, Kh.transpose(0, 1, 3, 2))                   # [B,H,J,K]
    Pm, A = bsb_fwd(S, mask_bias, scale, cfg.p_attn, cfg.seed, sub(SITE_ATTN), cfg.batch_offset)
    C = np.matmul(A, V).transpose(0, 2, 1, 3).reshape(B, J, I)
    Yo = _lin(C, prm["Wo"])
    Y, xhat, rstd = bdrln_fwd(Yo, prm["bo"], X, prm["g"], prm["be"], cfg.ln_eps, cfg.p_hidden,
                              cfg.seed, sub(SITE_ATTN_OUT), cfg.batch_offset)
    saved = dict(Q=Q, K=Kh, V=V, KV=KV, S=S, P=Pm, A=A, C=C, Yo=Yo, xhat=xhat, rstd=rstd, Y=Y)
    return Y, saved


def cross_attention_backward(dY, X, Mem, prm, H, cfg: Cfg, saved):
    """Returns (dX, dMem, grads) with grads keyed Wq, Wkv, Wo, bq, bkv, bo, g, be (sums over
    the local batch)."""
    dY, X, Mem = _f(dY), _f(X), _f(Mem)
    B, J, I = X.shape
    K = Mem.shape[1]
    P = I // H
    scale = 1.0 / np.sqrt(P)
    sub = lambda site: philox.subsequence(cfg.layer_id, site)   # noqa: E731
    sv = saved
    dz, dYo, dg, dbe, dbo = bdrln_bwd(dY, sv["xhat"], sv["rstd"], prm["g"], cfg.p_hidden,
                                      cfg.seed, sub(SITE_ATTN_OUT), cfg.batch_offset)
    dC = np.matmul(dYo, _f(prm["Wo"]))
    dWo = np.einsum("bji,bjk->ik", dYo, sv["C"])
    dCbh = dC.reshape(B, J, H, P).transpose(0, 2, 1, 3)
    dA = np.matmul(dCbh, sv["V"].transpose(0, 1, 3, 2))
    dV = np.matmul(sv["A"].transpose(0, 1, 3, 2), dCbh)          # [B,H,K,P]
    dS = bsb_bwd(dA, sv["P"], scale, cfg.p_attn, cfg.seed, sub(SITE_ATTN), cfg.batch_offset)
    dQ = np.matmul(dS, sv["K"])                                  # [B,H,J,P]
    dK = np.matmul(dS.transpose(0, 1, 3, 2), sv["Q"])            # [B,H,K,P]
    dQf = dQ.transpose(0, 2, 1, 3).reshape(B, J, I)
    dKV = np.concatenate([dK.transpose(0, 2, 1, 3).reshape(B, K, I),
                          dV.transpose(0, 2, 1, 3).reshape(B, K, I)], axis=-1)
    dX = np.matmul(dQf, _f(prm["Wq"])) + dz
    dMem = np.matmul(dKV, _f(prm["Wkv"]))
    grads = dict(Wq=np.einsum("bjo,bji->oi", dQf, X), Wkv=np.einsum("bko,bki->oi", dKV, Mem),
                 Wo=dWo, bq=dQf.sum(axis=(0, 1)), bkv=dKV.sum(axis=(0, 1)), bo=dbo, g=dg, be=dbe)
    return dX, dMem, grads
