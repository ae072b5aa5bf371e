"""EncoderStack (paper_2007_00072_b200/stack.py): n layers through the C ABI sharing one
context and one temporaries buffer.

* fp32, config T, 3 layers with distinct parameters and dropout subsequences (layer_id i,
  DESIGN.md R5): output, input gradient and every layer's parameter gradients against the
  fp64 oracle chained layer by layer (1e-5 normwise, tol.py).
* bf16, config L, 2 layers: the stack reproduces, bit for bit, the same layers run as
  independent EncoderLayer objects (own context, own scratch) -- sharing the scratch and
  the context's workspaces changes nothing.
"""
import numpy as np
import pytest
import torch

from oracle import encoder as E
from synth import CONFIGS, SEED_WEIGHTS, make_inputs, make_params
from tol import assert_parity

pytestmark = pytest.mark.gpu

TDT = {"bf16": torch.bfloat16, "fp32": torch.float32}


def f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def _run_stack(dims, dtype, n, p, key_padding):
    from paper_2007_00072_b200.layer import LayerCfg
    from paper_2007_00072_b200.stack import EncoderStack
    prms = [make_params(dims, dtype, "parity", seed=SEED_WEIGHTS + i) for i in range(n)]
    inp = make_inputs(dims, dtype, key_padding=key_padding)
    cfg = LayerCfg(p_attn=p, p_hidden=p, p_ffn=p)
    st = EncoderStack(n, dims, dtype, cfg)
    st.set_params(prms)
    X = torch.tensor(inp["X"], device="cuda").to(TDT[dtype])
    dY = torch.tensor(inp["dY"], device="cuda").to(TDT[dtype])
    M = None if inp["mask_bias"] is None else torch.tensor(inp["mask_bias"], device="cuda")
    done = []
    Y = st.forward(X, M).clone()
    dX = st.backward(dY, on_layer_done=lambda i, _l: done.append(i)).clone()
    torch.cuda.synchronize()
    assert done == list(reversed(range(n)))
    return st, prms, inp, X, dY, M, Y, dX


def test_stack_fp32_vs_oracle():
    dims, n, p = CONFIGS["T"], 3, 0.1
    st, prms, inp, *_rest, Y, dX = _run_stack(dims, "fp32", n, p, key_padding=True)
    xs, svs = [inp["X"]], []
    for i in range(n):
        ocfg = E.Cfg(p_attn=p, p_hidden=p, p_ffn=p, layer_id=i)
        y, sv = E.encoder_layer_forward(xs[-1], prms[i], dims.H, ocfg, inp["mask_bias"])
        xs.append(y)
        svs.append(sv)
    assert_parity("Y", f64(Y), xs[-1], "fp32")
    g = inp["dY"]
    for i in reversed(range(n)):
        ocfg = E.Cfg(p_attn=p, p_hidden=p, p_ffn=p, layer_id=i)
        g, go, _ = E.encoder_layer_backward(g, xs[i], prms[i], dims.H, ocfg, svs[i])
        for name, ref in go.items():
            assert_parity(f"layer{i}.d{name}", f64(st.layers[i].grads[name]), ref, "fp32")
    assert_parity("dX", f64(dX), g, "fp32")


def test_stack_bf16_matches_independent_layers():
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    dims, n, p = CONFIGS["L"], 2, 0.1
    st, prms, _inp, X, dY, M, Y, dX = _run_stack(dims, "bf16", n, p, key_padding=False)
    x, layers = X, []
    for i in range(n):
        layer = EncoderLayer(dims, "bf16", LayerCfg(p_attn=p, p_hidden=p, p_ffn=p, layer_id=i))
        layer.set_params(prms[i])
        x = layer.forward(x, M)
        layers.append((layer, x))
    inputs = [X] + [y for _l, y in layers[:-1]]
    g = dY
    for i in reversed(range(n)):
        g = layers[i][0].backward(inputs[i], g)
    torch.cuda.synchronize()
    assert torch.equal(Y.view(torch.int16), x.view(torch.int16))
    assert torch.equal(dX.view(torch.int16), g.view(torch.int16))
    for i in range(n):
        assert torch.equal(st.layers[i].grad_flat, layers[i][0].grad_flat), f"layer {i} grads"
