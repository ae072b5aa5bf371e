"""encoder_layer_step_host (host buffers in, host buffers out, copies overlapped on the
context's copy streams) equals the device-buffer forward + backward, bitwise; also when the
call is captured in a CUDA graph and replayed."""
import numpy as np
import pytest
import torch

from synth import CONFIGS, Dims, make_inputs, make_params

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims,dtype", [(CONFIGS["T"], "fp32"),
                                        (Dims(B=2, J=512, H=2, P=64, U=512), "bf16")])
@pytest.mark.parametrize("graph", [False, True])
def test_step_host_matches_device_path(dims, dtype, graph):
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    prm = make_params(dims, dtype, "parity", weight_std=0.05)
    inp = make_inputs(dims, dtype)
    layer = EncoderLayer(dims, dtype, LayerCfg())
    layer.set_params(prm)
    X = torch.tensor(inp["X"], device="cuda").to(tdt)
    dY = torch.tensor(inp["dY"], device="cuda").to(tdt)
    Y_ref = layer.forward(X)
    dX_ref = layer.backward(X, dY)
    g_ref = layer.grad_flat.clone()
    torch.cuda.synchronize()

    Xh, dYh = X.cpu().pin_memory(), dY.cpu().pin_memory()
    Yh = torch.full_like(Xh, float("nan")).pin_memory()
    dXh = torch.full_like(Xh, float("nan")).pin_memory()
    Xd, dYd = torch.empty_like(X), torch.empty_like(dY)
    Yd, dXd = torch.empty_like(X), torch.empty_like(X)
    layer.grad_flat.zero_()
    if graph:
        layer.step_host(Xh, dYh, Yh, dXh, Xd, dYd, Yd, dXd)   # warm-up outside capture
        torch.cuda.synchronize()
        Yh.fill_(float("nan"))
        dXh.fill_(float("nan"))
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            layer.step_host(Xh, dYh, Yh, dXh, Xd, dYd, Yd, dXd)
        g.replay()
    else:
        layer.step_host(Xh, dYh, Yh, dXh, Xd, dYd, Yd, dXd)
    torch.cuda.synchronize()
    assert torch.equal(Yh, Y_ref.cpu())
    assert torch.equal(dXh, dX_ref.cpu())
    assert torch.equal(layer.grad_flat, g_ref)
