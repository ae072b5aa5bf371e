"""Pins of the encoder-decoder (cross) attention oracle (oracle/encoder.py,
cross_attention_*):
  * p = 0: equals torch.nn.MultiheadAttention (query = X, key = value = memory; in_proj =
    [W^Q; W^K; W^V] with our stacked [W^K; W^V]) + residual + LayerNorm in fp64, forward and
    (autograd) backward, with and without a key-padding bias, for J != K;
  * with dropout: the same torch graph with the oracle's Philox masks injected at both sites;
  * central finite differences of the whole sublayer on a tiny shape."""
import numpy as np
import pytest
import torch

from oracle import encoder as E
from oracle import philox

RNG = np.random.default_rng(7)


def _params(I, std=0.3):
    r = lambda *s: RNG.standard_normal(s) * std  # noqa: E731
    return {"Wq": r(I, I), "Wkv": r(2 * I, I), "Wo": r(I, I), "bq": r(I) * 0.3,
            "bkv": r(2 * I) * 0.3, "bo": r(I) * 0.3, "g": 1 + r(I) * 0.3, "be": r(I) * 0.3}


def _torch_ref(X, Mem, prm, H, mask_bias, cfg, drop):
    """fp64 torch: MHA (batch_first) + dropout + residual + LayerNorm (post-LN)."""
    B, J, I = X.shape
    K = Mem.shape[1]
    P = I // H
    t = lambda a: torch.tensor(a, dtype=torch.float64, requires_grad=True)  # noqa: E731
    tX, tM = t(X), t(Mem)
    W = {k: t(v) for k, v in prm.items()}
    q = tX @ W["Wq"].T + W["bq"]
    kv = tM @ W["Wkv"].T + W["bkv"]
    k, v = kv[..., :I], kv[..., I:]
    sh = lambda a, L: a.reshape(B, L, H, P).transpose(1, 2)  # noqa: E731
    s = sh(q, J) @ sh(k, K).transpose(-1, -2) / np.sqrt(P)
    if mask_bias is not None:
        s = s + torch.tensor(mask_bias)[:, None, None, :]
    a = torch.softmax(s, -1)
    if drop:
        keep = philox.keep_mask_tensor((B, H, J, K), cfg.batch_offset, cfg.p_attn, cfg.seed,
                                       philox.subsequence(cfg.layer_id, 0))
        a = a * torch.tensor(keep) * philox.dropout_scale(cfg.p_attn)
    c = (a @ sh(v, K)).transpose(1, 2).reshape(B, J, I)
    yo = c @ W["Wo"].T + W["bo"]
    if drop:
        keep1 = philox.keep_mask_tensor((B, J, I), cfg.batch_offset, cfg.p_hidden, cfg.seed,
                                        philox.subsequence(cfg.layer_id, 1))
        yo = yo * torch.tensor(keep1) * philox.dropout_scale(cfg.p_hidden)
    y = torch.nn.functional.layer_norm(tX + yo, (I,), W["g"], W["be"], eps=cfg.ln_eps)
    return y, tX, tM, W


@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("drop", [False, True])
def test_cross_attention_matches_torch(masked, drop):
    B, J, K, H, P = 2, 5, 7, 2, 4
    I = H * P
    X = RNG.standard_normal((B, J, I))
    Mem = RNG.standard_normal((B, K, I))
    prm = _params(I)
    mb = None
    if masked:
        mb = np.zeros((B, K))
        mb[0, 5:] = -10000.0
    p = 0.2 if drop else 0.0
    cfg = E.Cfg(p_attn=p, p_hidden=p, p_ffn=p, layer_id=2, batch_offset=1)
    Y, sv = E.cross_attention_forward(X, Mem, prm, H, cfg, mb)
    dY = RNG.standard_normal(Y.shape)
    dX, dMem, g = E.cross_attention_backward(dY, X, Mem, prm, H, cfg, sv)
    y, tX, tM, W = _torch_ref(X, Mem, prm, H, mb, cfg, drop)
    y.backward(torch.tensor(dY))
    np.testing.assert_allclose(Y, y.detach().numpy(), rtol=1e-10, atol=1e-10)
    np.testing.assert_allclose(dX, tX.grad.numpy(), rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(dMem, tM.grad.numpy(), rtol=1e-9, atol=1e-9)
    for k in prm:
        np.testing.assert_allclose(g[k], W[k].grad.numpy(), rtol=1e-9, atol=1e-9, err_msg=k)


def test_cross_attention_finite_differences():
    B, J, K, H, P = 1, 3, 5, 2, 2
    I = H * P
    X = RNG.standard_normal((B, J, I))
    Mem = RNG.standard_normal((B, K, I))
    prm = _params(I)
    cfg = E.Cfg(p_attn=0.3, p_hidden=0.3, p_ffn=0.0)
    w = RNG.standard_normal((B, J, I))
    f = lambda X_, M_, p_: float((E.cross_attention_forward(X_, M_, p_, H, cfg)[0] * w).sum())  # noqa
    Y, sv = E.cross_attention_forward(X, Mem, prm, H, cfg)
    dX, dMem, g = E.cross_attention_backward(w, X, Mem, prm, H, cfg, sv)
    eps = 1e-6
    for _ in range(12):
        i = tuple(RNG.integers(0, s) for s in Mem.shape)
        Mp, Mm = Mem.copy(), Mem.copy()
        Mp[i] += eps
        Mm[i] -= eps
        assert abs((f(X, Mp, prm) - f(X, Mm, prm)) / (2 * eps) - dMem[i]) < 1e-6
    for name in ("Wkv", "Wq", "bkv"):
        for _ in range(6):
            i = tuple(RNG.integers(0, s) for s in prm[name].shape)
            pp = {k: v.copy() for k, v in prm.items()}
            pm = {k: v.copy() for k, v in prm.items()}
            pp[name][i] += eps
            pm[name][i] -= eps
            assert abs((f(X, Mem, pp) - f(X, Mem, pm)) / (2 * eps) - g[name][i]) < 1e-6
