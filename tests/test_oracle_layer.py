"""Whole-layer pins for oracle/encoder.py (CPU only).

* p = 0: the layer equals torch.nn.TransformerEncoderLayer (post-LN, batch_first) in
  fp64, forward and autograd backward ("Special case reducing to a
  library routine").
* p > 0: the layer equals the same torch layer with the oracle's Philox keep masks
  injected at torch's own four dropout sites; this pins WHERE the dropouts sit.
* central finite differences pin the analytic backward on the tiny config.
"""
import contextlib

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from oracle import encoder as E
from oracle import philox
from synth import CONFIGS, Dims, make_inputs, make_params

ACTS = {
    E.ACT_RELU: "relu",
    E.ACT_GELU_ERF: "gelu",
    E.ACT_GELU_TANH: (lambda x: F.gelu(x, approximate="tanh")),
}


def _torch_layer(prm, dims, act, eps):
    layer = torch.nn.TransformerEncoderLayer(
        d_model=dims.I, nhead=dims.H, dim_feedforward=dims.U, dropout=0.0,
        activation=ACTS[act], batch_first=True, norm_first=False, layer_norm_eps=eps,
        dtype=torch.float64)
    t = lambda a: torch.tensor(np.asarray(a, np.float64))  # noqa: E731
    with torch.no_grad():
        layer.self_attn.in_proj_weight.copy_(t(prm["Wqkv"]))
        layer.self_attn.in_proj_bias.copy_(t(prm["bqkv"]))
        layer.self_attn.out_proj.weight.copy_(t(prm["Wo"]))
        layer.self_attn.out_proj.bias.copy_(t(prm["bo"]))
        layer.linear1.weight.copy_(t(prm["W1"]))
        layer.linear1.bias.copy_(t(prm["b1"]))
        layer.linear2.weight.copy_(t(prm["W2"]))
        layer.linear2.bias.copy_(t(prm["b2"]))
        layer.norm1.weight.copy_(t(prm["g1"]))
        layer.norm1.bias.copy_(t(prm["be1"]))
        layer.norm2.weight.copy_(t(prm["g2"]))
        layer.norm2.bias.copy_(t(prm["be2"]))
    layer.train()
    return layer


def _torch_grads(layer):
    sa = layer.self_attn
    return dict(Wqkv=sa.in_proj_weight.grad, bqkv=sa.in_proj_bias.grad,
                Wo=sa.out_proj.weight.grad, bo=sa.out_proj.bias.grad,
                W1=layer.linear1.weight.grad, b1=layer.linear1.bias.grad,
                W2=layer.linear2.weight.grad, b2=layer.linear2.bias.grad,
                g1=layer.norm1.weight.grad, be1=layer.norm1.bias.grad,
                g2=layer.norm2.weight.grad, be2=layer.norm2.bias.grad)


class _Inject(torch.nn.Module):
    """Replaces an nn.Dropout: multiplies by a fixed (keep * scale) tensor."""

    def __init__(self, m):
        super().__init__()
        self.m = m

    def forward(self, x):
        return x * self.m


@contextlib.contextmanager
def _inject_attention_dropout(layer, m_attn, p):
    """torch's MHA applies F.dropout to the attention weights [B*H, J, K] on its
    need_weights=True path (torch/nn/functional.py multi_head_attention_forward)."""
    sa = layer.self_attn
    sa.dropout = p
    orig_fwd = sa.forward
    orig_dropout = F.dropout

    def fwd(*a, **k):
        k["need_weights"] = True
        k["average_attn_weights"] = False
        return orig_fwd(*a, **k)

    def drop(x, p=0.5, training=True, inplace=False):
        assert x.shape == m_attn.shape
        return x * m_attn

    sa.forward = fwd
    F.dropout = drop
    try:
        yield
    finally:
        F.dropout = orig_dropout
        sa.forward = orig_fwd


def _run_both(dims, act, key_padding, p, seed=2007000072, batch_offset=0, eps=1e-5,
              causal=False):
    prm = make_params(dims, "fp32", "parity", weight_std=0.2)
    inp = make_inputs(dims, "fp32", key_padding=key_padding)
    cfg = E.Cfg(p_attn=p, p_hidden=p, p_ffn=p, seed=seed, layer_id=3,
                batch_offset=batch_offset, ln_eps=eps, act=act, causal=causal)
    Y, saved = E.encoder_layer_forward(inp["X"], prm, dims.H, cfg, inp["mask_bias"])
    dX, grads, _ = E.encoder_layer_backward(inp["dY"], inp["X"], prm, dims.H, cfg, saved)

    layer = _torch_layer(prm, dims, act, eps)
    X = torch.tensor(inp["X"].astype(np.float64), requires_grad=True)
    kpm = None if inp["mask_bias"] is None else torch.tensor(inp["mask_bias"].astype(np.float64))
    ctx = contextlib.nullcontext()
    if p > 0:
        B, J, H, I, U = dims.B, dims.J, dims.H, dims.I, dims.U
        s = philox.dropout_scale(p)
        mk = lambda shape, site: torch.tensor(  # noqa: E731
            philox.keep_mask_tensor(shape, batch_offset, p, seed, philox.subsequence(3, site)) * s)
        layer.dropout1 = _Inject(mk((B, J, I), E.SITE_ATTN_OUT))
        layer.dropout = _Inject(mk((B, J, U), E.SITE_FFN))
        layer.dropout2 = _Inject(mk((B, J, I), E.SITE_FFN_OUT))
        ctx = _inject_attention_dropout(layer, mk((B, H, J, J), E.SITE_ATTN).reshape(B * H, J, J), p)
    src_mask = None
    if causal:   # torch's own "square subsequent" mask: -inf above the diagonal
        src_mask = torch.nn.Transformer.generate_square_subsequent_mask(
            dims.J, dtype=torch.float64)
    with ctx:
        Yt = layer(X, src_mask=src_mask, src_key_padding_mask=kpm)
    Yt.backward(torch.tensor(inp["dY"].astype(np.float64)))
    return (Y, dX, grads), (Yt.detach().numpy(), X.grad.numpy(),
                            {k: v.numpy() for k, v in _torch_grads(layer).items()})


def _assert_close(a, b, tol=1e-10):
    scale = max(np.abs(b).max(), 1e-30)
    assert np.abs(a - b).max() / scale < tol


@pytest.mark.parametrize("act", [E.ACT_RELU, E.ACT_GELU_ERF, E.ACT_GELU_TANH])
@pytest.mark.parametrize("key_padding", [False, True])
def test_layer_equals_torch_transformer_encoder_layer_p0(act, key_padding):
    dims = CONFIGS["T"]
    (Y, dX, g), (Yt, dXt, gt) = _run_both(dims, act, key_padding, 0.0)
    _assert_close(Y, Yt)
    _assert_close(dX, dXt)
    for k in g:
        _assert_close(g[k], gt[k])


@pytest.mark.parametrize("act", [E.ACT_RELU, E.ACT_GELU_ERF])
def test_layer_dropout_placement_matches_torch_sites(act):
    dims = CONFIGS["T"]
    (Y, dX, g), (Yt, dXt, gt) = _run_both(dims, act, True, 0.1, batch_offset=5)
    _assert_close(Y, Yt)
    _assert_close(dX, dXt)
    for k in g:
        _assert_close(g[k], gt[k])


@pytest.mark.parametrize("key_padding", [False, True])
@pytest.mark.parametrize("p", [0.0, 0.1])
def test_layer_causal_equals_torch(key_padding, p):
    """Causal masking (R22) against torch's layer with its
    square-subsequent mask, with and without key padding and dropout."""
    dims = CONFIGS["T"]
    (Y, dX, g), (Yt, dXt, gt) = _run_both(dims, E.ACT_GELU_ERF, key_padding, p, causal=True,
                                          batch_offset=2)
    _assert_close(Y, Yt)
    _assert_close(dX, dXt)
    for k in g:
        _assert_close(g[k], gt[k])


def test_causal_softmax_rows():
    """Row j of a causal P has j+1 nonzeros summing to 1; row 0 is the one-hot e_0."""
    rng = np.random.default_rng(5)
    S = rng.standard_normal((2, 3, 9, 9))
    Pm, _ = E.bsb_fwd(S, None, 0.5, 0.0, 1, 0, causal=True)
    assert np.allclose(Pm.sum(-1), 1.0, atol=1e-12)
    assert np.all(np.triu(Pm, 1) == 0.0)
    assert np.allclose(Pm[..., 0, 0], 1.0)
    assert np.all(Pm[..., np.tril(np.ones((9, 9), bool))] > 0)


def test_degenerate_single_head():
    dims = Dims(B=2, J=8, H=1, P=16, U=32)      # H = 1, P = I
    (Y, dX, g), (Yt, dXt, gt) = _run_both(dims, E.ACT_GELU_ERF, False, 0.0)
    _assert_close(Y, Yt)
    _assert_close(dX, dXt)


def test_finite_differences_tiny_with_dropout():
    """Central differences, step 1e-5, 64 random coordinates per tensor, masks fixed
    (SPEC.md:465-473 protocol); relative error < 1e-6."""
    dims = CONFIGS["T"]
    prm = make_params(dims, "fp32", "parity", weight_std=0.2)
    prm = {k: v.astype(np.float64) for k, v in prm.items()}
    inp = make_inputs(dims, "fp32", key_padding=True)
    X = inp["X"].astype(np.float64)
    dY = inp["dY"].astype(np.float64)
    cfg = E.Cfg(p_attn=0.1, p_hidden=0.1, p_ffn=0.1, act=E.ACT_GELU_ERF, layer_id=1)
    Y, saved = E.encoder_layer_forward(X, prm, dims.H, cfg, inp["mask_bias"])
    dX, grads, _ = E.encoder_layer_backward(dY, X, prm, dims.H, cfg, saved)

    def loss(Xv, pv):
        Yv, _ = E.encoder_layer_forward(Xv, pv, dims.H, cfg, inp["mask_bias"])
        return float((Yv * dY).sum())

    rng = np.random.default_rng(3)
    h = 1e-5
    targets = [("X", X, dX)] + [(k, prm[k], grads[k]) for k in prm]
    for name, arr, ana in targets:
        flat = arr.reshape(-1)
        idx = rng.choice(flat.size, size=min(64, flat.size), replace=False)
        num = np.empty(idx.size)
        for t, i in enumerate(idx):
            old = flat[i]
            flat[i] = old + h
            lp = loss(X, prm)
            flat[i] = old - h
            lm = loss(X, prm)
            flat[i] = old
            num[t] = (lp - lm) / (2 * h)
        a = ana.reshape(-1)[idx]
        err = np.abs(num - a).max() / max(np.abs(a).max(), 1e-12)
        assert err < 1e-6, (name, err)


def test_data_parallel_partition_reproduces_global_batch():
    """Rank r owns global batch rows [r*Bl, (r+1)*Bl) with batch_offset = r*Bl: the
    per-rank outputs are slices of the global run and the per-rank gradient SUMS add up
    to the global gradients."""
    dims = Dims(B=4, J=8, H=2, P=4, U=16)
    prm = make_params(dims, "fp32", "parity", weight_std=0.2)
    inp = make_inputs(dims, "fp32", key_padding=True)
    cfg = E.Cfg(p_attn=0.2, p_hidden=0.2, p_ffn=0.2, layer_id=2)
    Y, sv = E.encoder_layer_forward(inp["X"], prm, dims.H, cfg, inp["mask_bias"])
    dX, g, _ = E.encoder_layer_backward(inp["dY"], inp["X"], prm, dims.H, cfg, sv)
    acc = {k: 0.0 for k in g}
    for r in range(2):
        sl = slice(2 * r, 2 * r + 2)
        c = E.Cfg(**{**cfg.__dict__, "batch_offset": 2 * r})
        Yr, svr = E.encoder_layer_forward(inp["X"][sl], prm, dims.H, c, inp["mask_bias"][sl])
        dXr, gr, _ = E.encoder_layer_backward(inp["dY"][sl], inp["X"][sl], prm, dims.H, c, svr)
        assert np.allclose(Yr, Y[sl], atol=1e-12)
        assert np.allclose(dXr, dX[sl], atol=1e-12)
        for k in g:
            acc[k] = acc[k] + gr[k]
    for k in g:
        assert np.allclose(acc[k], g[k], atol=1e-11)
