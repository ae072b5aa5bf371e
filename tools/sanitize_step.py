"""One encoder-layer forward + backward at config T (fp32) and at a small bf16 shape on the
product path (tcgen05 weight contractions with the fused FFN epilogues, fused score
kernels, per-(b,h) attention contractions): the workload tests/test_gpu_sanitizer.py runs
under compute-sanitizer (memcheck / racecheck / synccheck / initcheck)."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2007_00072_b200.layer import EncoderLayer, LayerCfg
    from synth import CONFIGS, Dims, make_inputs, make_params
    for dims, dtype in ((CONFIGS["T"], "fp32"), (Dims(B=1, J=512, H=2, P=64, U=512), "bf16")):
        prm = make_params(dims, dtype, "parity", weight_std=0.1)
        inp = make_inputs(dims, dtype, key_padding=True)
        tdt = torch.float32 if dtype == "fp32" else torch.bfloat16
        layer = EncoderLayer(dims, dtype, LayerCfg())
        if os.environ.get("ENC_SANITIZE_SINGLE_CTA") == "1":
            from paper_2007_00072_b200 import ops
            ops.enc_set_option(layer.ctx, ops.OPT_GEMM_PAIR, 0)
        layer.set_params(prm)
        X = torch.tensor(inp["X"], device="cuda").to(tdt)
        dY = torch.tensor(inp["dY"], device="cuda").to(tdt)
        M = torch.tensor(inp["mask_bias"], device="cuda")
        layer.forward(X, M)
        layer.backward(X, dY)
        torch.cuda.synchronize()
    print("sanitize_step done", flush=True)


if __name__ == "__main__":
    main()
