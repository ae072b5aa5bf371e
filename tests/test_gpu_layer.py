"""Whole-layer parity: encoder_layer_forward / encoder_layer_backward through the C ABI vs
the fp64 oracle on the same seeded inputs (configs T, a small bf16 case, and the paper's
BERT-large layer L at full size)."""
import numpy as np
import pytest
import torch

from oracle import encoder as E
from synth import CONFIGS, Dims, make_inputs, make_params
from tol import assert_parity, errors

pytestmark = pytest.mark.gpu

ACT = {"gelu": E.ACT_GELU_ERF, "gelu_tanh": E.ACT_GELU_TANH, "relu": E.ACT_RELU}
TDT = {"bf16": torch.bfloat16, "fp32": torch.float32}


def _run(dims, dtype, act, key_padding, p=0.1, batch_offset=0, layer_id=0, weight_std=0.02):
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    prm = make_params(dims, dtype, "parity", weight_std=weight_std)
    inp = make_inputs(dims, dtype, key_padding=key_padding)
    cfg = LayerCfg(p_attn=p, p_hidden=p, p_ffn=p, act=act, layer_id=layer_id,
                   batch_offset=batch_offset)
    layer = EncoderLayer(dims, dtype, cfg)
    layer.set_params(prm)
    X = torch.tensor(inp["X"], device="cuda").to(TDT[dtype])
    dY = torch.tensor(inp["dY"], device="cuda").to(TDT[dtype])
    M = None if inp["mask_bias"] is None else torch.tensor(inp["mask_bias"], device="cuda")
    Y = layer.forward(X, M)
    dX = layer.backward(X, dY)
    torch.cuda.synchronize()
    ocfg = E.Cfg(p_attn=p, p_hidden=p, p_ffn=p, act=ACT[act], layer_id=layer_id,
                 batch_offset=batch_offset)
    Yo, sv = E.encoder_layer_forward(inp["X"], prm, dims.H, ocfg, inp["mask_bias"])
    dXo, go, inter = E.encoder_layer_backward(inp["dY"], inp["X"], prm, dims.H, ocfg, sv)
    f = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
    gpu = {"Y": f(Y), "dX": f(dX)}
    ref = {"Y": Yo, "dX": dXo}
    for n in go:
        gpu["d" + n] = f(layer.grads[n])
        ref["d" + n] = go[n]
    sv_gpu = layer.saved_views()
    for n in ("Q", "K", "V", "P", "A", "C", "X1", "xhat1", "h", "A1", "xhat2", "rstd1", "rstd2"):
        gpu["saved." + n] = f(sv_gpu[n])
        ref["saved." + n] = sv[n]
    return gpu, ref


@pytest.mark.parametrize("act", ["gelu", "relu", "gelu_tanh"])
def test_layer_T_fp32(act):
    gpu, ref = _run(CONFIGS["T"], "fp32", act, key_padding=True, weight_std=0.2)
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "fp32")


def test_layer_T_fp32_batch_offset_and_layer_id():
    gpu, ref = _run(CONFIGS["T"], "fp32", "gelu", key_padding=False, batch_offset=6,
                    layer_id=7, weight_std=0.2)
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "fp32")


def test_layer_T_fp32_no_dropout():
    gpu, ref = _run(CONFIGS["T"], "fp32", "gelu", key_padding=True, p=0.0, weight_std=0.2)
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "fp32")


def test_layer_small_bf16():
    dims = Dims(B=2, J=64, H=4, P=16, U=256)
    gpu, ref = _run(dims, "bf16", "gelu", key_padding=True, weight_std=0.06)
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "bf16")


def test_layer_L_bf16_full():
    """The paper's BERT-large layer (B=8, J=K=512, H=16, P=64, I=1024, U=4096) at full
    size, bf16 with fp32 accumulation/statistics, vs the fp64 oracle on the same inputs."""
    gpu, ref = _run(CONFIGS["L"], "bf16", "gelu", key_padding=False)
    report = {n: errors(gpu[n], ref[n]) for n in gpu}
    for n, e in sorted(report.items()):
        print(f"{n:14s} max/rms {e['max_over_rms']:.3e} mean_rel {e['mean_rel']:.3e}")
    for n in gpu:
        assert_parity(n, gpu[n], ref[n], "bf16")
