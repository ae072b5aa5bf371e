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


@pytest.mark.parametrize("dims,dtype", [(CONFIGS["T"], "fp32"),
                                        (Dims(B=2, J=512, H=2, P=64, U=512), "bf16")])
def test_step_host_pipelined_matches_device_path(dims, dtype):
    """Three pipelined steps on different inputs (input prefetch on the copy-in stream,
    output copies on the copy-out stream, double-buffered device buffers) give each step's
    device-path Y and dX bitwise, and the last step's gradients."""
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    prm = make_params(dims, dtype, "parity", weight_std=0.05)
    layer = EncoderLayer(dims, dtype, LayerCfg())
    layer.set_params(prm)
    base = make_inputs(dims, dtype)
    steps = 3
    Xs = [torch.tensor(base["X"], device="cuda").to(tdt) * (1 + 0.25 * s) for s in range(steps)]
    dYs = [torch.tensor(base["dY"], device="cuda").to(tdt) * (1 - 0.2 * s) for s in range(steps)]
    refs = []
    for s in range(steps):
        Y = layer.forward(Xs[s]).clone()
        dX = layer.backward(Xs[s], dYs[s]).clone()
        refs.append((Y.cpu(), dX.cpu()))
    g_ref = layer.grad_flat.clone()
    torch.cuda.synchronize()

    Xh = [x.cpu().pin_memory() for x in Xs]
    dYh = [d.cpu().pin_memory() for d in dYs]
    Yh = [torch.full_like(Xh[0], float("nan")).pin_memory() for _ in range(steps)]
    dXh = [torch.full_like(Xh[0], float("nan")).pin_memory() for _ in range(steps)]
    Xd = [torch.empty_like(Xs[0]) for _ in range(2)]
    dYd = [torch.empty_like(Xs[0]) for _ in range(2)]
    Yd = [torch.empty_like(Xs[0]) for _ in range(2)]
    dXd = [torch.empty_like(Xs[0]) for _ in range(2)]
    layer.grad_flat.zero_()
    layer.prefetch_inputs(Xh[0], dYh[0], Xd[0], dYd[0])
    for s in range(steps):
        a, b = s & 1, (s + 1) & 1
        nxt = s + 1 < steps
        layer.step_host_pipelined(Xd[a], dYd[a], Yd[a], dXd[a], Yh[s],
                                  Xh[s + 1] if nxt else None, dYh[s + 1] if nxt else None,
                                  Xd[b], dYd[b],
                                  dXd[b] if s else None, dXh[s - 1] if s else None)
    dXh[steps - 1].copy_(dXd[(steps - 1) & 1], non_blocking=True)
    torch.cuda.synchronize()
    for s in range(steps):
        assert torch.equal(Yh[s], refs[s][0]), s
        assert torch.equal(dXh[s], refs[s][1]), s
    assert torch.equal(layer.grad_flat, g_ref)


def test_step_host_pipelined_rejects_aliased_prefetch():
    from paper_2007_00072_b200._abi import EncError
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    dims = CONFIGS["T"]
    layer = EncoderLayer(dims, "fp32", LayerCfg())
    layer.set_params(make_params(dims, "fp32", "parity"))
    X = torch.zeros((dims.B, dims.J, dims.I), device="cuda")
    h = X.cpu().pin_memory()
    with pytest.raises(EncError):
        layer.step_host_pipelined(X, X.clone(), X.clone(), X.clone(), h, h, h, X, X.clone())
