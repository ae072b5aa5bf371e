"""bf16-storage model of the layer (test infrastructure, R14): the fp64 oracle's
per-operator functions (oracle/encoder.py) chained exactly as the full-precision oracle
chains them, but with every tensor the bf16 GPU path STORES rounded to bf16 (round to
nearest even) before its consumers read it.  It contains no arithmetic of its own beyond
that rounding and the plain contractions of the oracle.

Its distance to the full-precision oracle is the error that bf16 storage alone causes
(the conditioning of the layer), which bounds what any bf16 implementation can reach end
to end; the GPU's end-to-end error is asserted against it in tests/test_gpu_layer.py and
smoke().  Storage points (the default bf16 path, include/encoder.h): QKV (bias added before
rounding), P, C, Yo, X1, xhat1, h, A1, Y2, Y, xhat2; backward dz2, dY2, dh, dX1, dz1, dYo,
dC, dV, dS, dQ, dK, dX.  Kept in fp32 (never stored): the scores S and their gradient dA
(TMEM), A = dropout(P) (applied on load), dA1 (TMEM of the fused Linear2-dX + BAD-bwd)."""
import numpy as np

from oracle import encoder as E
from oracle import philox
from synth import bf16_round


def r(a):
    return bf16_round(np.asarray(a, np.float32)).astype(np.float64)


def layer(X, prm, H, cfg, mask_bias=None, dY=None):
    """Forward (and backward if dY is given) with bf16 storage.  Returns a dict with the
    keys of tests/test_gpu_layer._end_to_end: Y, dX, d<param>, saved.<name>."""
    X = np.asarray(X, np.float64)
    W = {k: np.asarray(v, np.float64) for k, v in prm.items()}
    B, J, I = X.shape
    P = I // H
    sc = 1.0 / np.sqrt(P)
    sub = lambda site: philox.subsequence(cfg.layer_id, site)  # noqa: E731
    seed, boff = cfg.seed, cfg.batch_offset
    QKV = r(X @ W["Wqkv"].T + W["bqkv"])
    Q, K, V = E.aib_fwd(QKV, np.zeros(3 * I), H, P)
    S = Q @ K.transpose(0, 1, 3, 2)
    Pm, A = E.bsb_fwd(S, mask_bias, sc, cfg.p_attn, seed, sub(0), boff, causal=cfg.causal)
    Pm = r(Pm)
    keep0 = philox.keep_mask_tensor(Pm.shape, boff, cfg.p_attn, seed, sub(0))
    A = np.where(keep0, Pm * philox.dropout_scale(cfg.p_attn), 0.0)
    C = r((A @ V).transpose(0, 2, 1, 3).reshape(B, J, I))
    Yo = r(C @ W["Wo"].T)
    X1, xh1, r1 = E.bdrln_fwd(Yo, W["bo"], X, W["g1"], W["be1"], cfg.ln_eps, cfg.p_hidden, seed,
                              sub(1), boff)
    X1, xh1 = r(X1), r(xh1)
    h = r(X1 @ W["W1"].T + W["b1"])
    _, A1 = E.bad_fwd(h, np.zeros_like(W["b1"]), cfg.act, cfg.p_ffn, seed, sub(2), boff)
    A1 = r(A1)
    Y2 = r(A1 @ W["W2"].T)
    Y, xh2, r2 = E.bdrln_fwd(Y2, W["b2"], X1, W["g2"], W["be2"], cfg.ln_eps, cfg.p_hidden, seed,
                             sub(3), boff)
    Y, xh2 = r(Y), r(xh2)
    out = {"Y": Y}
    for n, v in (("Q", Q), ("K", K), ("V", V), ("P", Pm), ("C", C), ("X1", X1), ("xhat1", xh1),
                 ("h", h), ("A1", A1), ("xhat2", xh2), ("rstd1", r1), ("rstd2", r2)):
        out["saved." + n] = v
    if dY is None:
        return out
    dY = np.asarray(dY, np.float64)
    dz2, dY2, dg2, dbe2, db2 = E.bdrln_bwd(dY, xh2, r2, W["g2"], cfg.p_hidden, seed, sub(3), boff)
    dz2, dY2 = r(dz2), r(dY2)
    dA1 = dY2 @ W["W2"]
    dW2 = np.einsum("bji,bju->iu", dY2, A1)
    dh, db1 = E.bad_bwd(dA1, h, cfg.act, cfg.p_ffn, seed, sub(2), boff)
    dh = r(dh)
    dX1 = r(dh @ W["W1"] + dz2)
    dW1 = np.einsum("bju,bji->ui", dh, X1)
    dz1, dYo, dg1, dbe1, dbo = E.bdrln_bwd(dX1, xh1, r1, W["g1"], cfg.p_hidden, seed, sub(1),
                                           boff)
    dz1, dYo = r(dz1), r(dYo)
    dC = r(dYo @ W["Wo"])
    dWo = np.einsum("bji,bjk->ik", dYo, C)
    dCbh = dC.reshape(B, J, H, P).transpose(0, 2, 1, 3)
    dA = dCbh @ V.transpose(0, 1, 3, 2)
    dV = r(A.transpose(0, 1, 3, 2) @ dCbh)
    dS = r(E.bsb_bwd(dA, Pm, sc, cfg.p_attn, seed, sub(0), boff))
    dQ = r(dS @ K)
    dK = r(dS.transpose(0, 1, 3, 2) @ Q)
    dQKV, dbqkv = E.aib_bwd(dQ, dK, dV)
    dX = r(dQKV @ W["Wqkv"] + dz1)
    dWqkv = np.einsum("bjo,bji->oi", dQKV, X)
    out["dX"] = dX
    for n, v in (("Wqkv", dWqkv), ("bqkv", dbqkv), ("Wo", dWo), ("bo", dbo), ("W1", dW1),
                 ("b1", db1), ("W2", dW2), ("b2", db2), ("g1", dg1), ("be1", dbe1), ("g2", dg2),
                 ("be2", dbe2)):
        out["d" + n] = v
    return out


def cross_attention(X, Mem, prm, H, cfg, mask_bias=None, dY=None):
    """The encoder-decoder attention sublayer (oracle cross_attention_*) with bf16 storage at
    the CUDA path's storage points: Q, KV, S, P, A, C, Yo, Y, xhat; dz, dYo, dC, dA, dV, dS,
    dQ, dK, dX, dMem (the unfused attention path stores S, A, dA)."""
    X, Mem = np.asarray(X, np.float64), np.asarray(Mem, np.float64)
    W = {k: np.asarray(v, np.float64) for k, v in prm.items()}
    B, J, I = X.shape
    K = Mem.shape[1]
    P = I // H
    sc = 1.0 / np.sqrt(P)
    sub = lambda site: philox.subsequence(cfg.layer_id, site)  # noqa: E731
    seed, boff = cfg.seed, cfg.batch_offset
    Qf = r(X @ W["Wq"].T + W["bq"])
    KV = r(Mem @ W["Wkv"].T + W["bkv"])
    Q = Qf.reshape(B, J, H, P).transpose(0, 2, 1, 3)
    Kh = KV[..., :I].reshape(B, K, H, P).transpose(0, 2, 1, 3)
    V = KV[..., I:].reshape(B, K, H, P).transpose(0, 2, 1, 3)
    S = r(Q @ Kh.transpose(0, 1, 3, 2))
    Pm, A = E.bsb_fwd(S, mask_bias, sc, cfg.p_attn, seed, sub(0), boff)
    Pm, A = r(Pm), r(A)
    C = r((A @ V).transpose(0, 2, 1, 3).reshape(B, J, I))
    Yo = r(C @ W["Wo"].T)
    Y, xh, rs = E.bdrln_fwd(Yo, W["bo"], X, W["g"], W["be"], cfg.ln_eps, cfg.p_hidden, seed,
                            sub(1), boff)
    Y, xh = r(Y), r(xh)
    out = {"Y": Y}
    if dY is None:
        return out
    dY = np.asarray(dY, np.float64)
    dz, dYo, dg, dbe, dbo = E.bdrln_bwd(dY, xh, rs, W["g"], cfg.p_hidden, seed, sub(1), boff)
    dz, dYo = r(dz), r(dYo)
    dC = r(dYo @ W["Wo"])
    dWo = np.einsum("bji,bjk->ik", dYo, C)
    dCbh = dC.reshape(B, J, H, P).transpose(0, 2, 1, 3)
    dA = r(dCbh @ V.transpose(0, 1, 3, 2))
    dV = r(A.transpose(0, 1, 3, 2) @ dCbh)
    dS = r(E.bsb_bwd(dA, Pm, sc, cfg.p_attn, seed, sub(0), boff))
    dQ = r(dS @ Kh)
    dK = r(dS.transpose(0, 1, 3, 2) @ Q)
    dQf = dQ.transpose(0, 2, 1, 3).reshape(B, J, I)
    dKV = np.concatenate([dK.transpose(0, 2, 1, 3).reshape(B, K, I),
                          dV.transpose(0, 2, 1, 3).reshape(B, K, I)], axis=-1)
    out["dX"] = r(dQf @ W["Wq"] + dz)
    out["dMem"] = r(dKV @ W["Wkv"])
    g = {"Wq": np.einsum("bjo,bji->oi", dQf, X), "Wkv": np.einsum("bko,bki->oi", dKV, Mem),
         "Wo": dWo, "bq": dQf.sum(axis=(0, 1)), "bkv": dKV.sum(axis=(0, 1)), "bo": dbo, "g": dg,
         "be": dbe}
    for n, v in g.items():
        out["d" + n] = v
    return out
