#!/usr/bin/env python
"""One eager layer step (forward + backward, config L, bf16, p = 0.1, GELU) bracketed by
cudaProfilerStart/Stop after warm-up, for `ncu --profile-from-start off` launch lists and
full captures of the current kernels.  --optimizer adds one AdamW update of the layer.
  ncu --profile-from-start off --metrics gpu__time_duration.sum,... python tools/one_step.py
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--optimizer", action="store_true")
    ap.add_argument("--config", default="L", choices=["L", "Bb"])
    ap.add_argument("--opt", action="append", default=[], metavar="KEY=VALUE",
                    help="enc_set_option on the layer context (include/encoder.h ENC_OPT_*)")
    a = ap.parse_args()
    import torch
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    from synth import CONFIGS, make_inputs, make_params
    dims = CONFIGS[a.config]
    layer = EncoderLayer(dims, "bf16", LayerCfg())
    layer.set_params(make_params(dims, "bf16", "bench"))
    from paper_2007_00072_b200 import ops
    ops.enc_set_option(layer.ctx, 3, 1)   # tune cuBLASLt in the warm-up steps (bench does too)
    for kv in a.opt:
        k, v = (int(x) for x in kv.split("="))
        ops.enc_set_option(layer.ctx, k, v)
    inp = make_inputs(dims, "bf16")
    X = torch.tensor(inp["X"], device="cuda").to(torch.bfloat16)
    dY = torch.tensor(inp["dY"], device="cuda").to(torch.bfloat16)
    if a.optimizer:
        layer.init_optimizer()
    for _ in range(3):
        layer.forward(X)
        layer.backward(X, dY)
        if a.optimizer:
            layer.optimizer_step()
    torch.cuda.synchronize()
    ops.enc_set_option(layer.ctx, 3, 0)
    torch.cuda.cudart().cudaProfilerStart()
    layer.forward(X)
    layer.backward(X, dY)
    if a.optimizer:
        layer.optimizer_step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
