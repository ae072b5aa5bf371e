import sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from paper_2007_00072_b200 import ops
from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
from synth import Dims, make_inputs, make_params
dims = Dims(B=2, J=512, H=2, P=64, U=512)
prm = make_params(dims, "bf16", "parity", weight_std=0.06)
inp = make_inputs(dims, "bf16", key_padding=True)
X = torch.tensor(inp["X"], device="cuda").to(torch.bfloat16)
dY = torch.tensor(inp["dY"], device="cuda").to(torch.bfloat16)
M = torch.tensor(inp["mask_bias"], device="cuda")
res = {}
for tag, opts in [("stacked", {}), ("sep", {12: 0}), ("sep_tc", {12: 0, 8: 1}), ("stacked_tc", {8: 1}), ("qk", {12: 1})]:
    layer = EncoderLayer(dims, "bf16", LayerCfg())
    for k, v in opts.items():
        ops.enc_set_option(layer.ctx, k, v)
    layer.set_params(prm)
    Y = layer.forward(X, M).float().clone()
    dX = layer.backward(X, dY).float().clone()
    torch.cuda.synchronize()
    res[tag] = (Y, dX, layer.bwd_views()["dQKV"].float().clone(), layer.grads["Wqkv"].clone())
for tag in res:
    Y, dX, dq, gw = res[tag]
    Y0, dX0, dq0, gw0 = res["stacked"]
    print(tag, "Y", (Y - Y0).abs().max().item(), "dQKV", (dq - dq0).abs().max().item(), "dX", (dX - dX0).abs().max().item(), "dW", (gw-gw0).abs().max().item(), "dXmax", dX0.abs().max().item())
