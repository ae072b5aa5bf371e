#!/usr/bin/env python
"""Time the attention contractions (enc_attn_gemm) at config L (B=8, H=16, J=K=512, P=64,
bf16) on the per-(b, h) streaming kernel and on the tiled kernel: L2 flushed before every
launch, CUDA events on the launching stream, median of --reps.  Under ncu use --reps 1."""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--B", type=int, default=8)
    ap.add_argument("--which", default="1,3,4,5")
    ap.add_argument("--bh", default="1,0")
    args = ap.parse_args()
    import torch
    from paper_2007_00072_b200 import ops
    B, H, J, P = args.B, 16, 512, 64
    dev = torch.device("cuda", 0)
    ctx = ops.Context(0)
    bf = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(0)
    big = torch.randn((B, H, J, J), device=dev, generator=g).to(bf)
    small = torch.randn((B, H, J, P), device=dev, generator=g).to(bf)
    out = torch.empty((B, H, J, P), device=dev, dtype=bf)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    names = {1: "AV", 3: "dV", 4: "dQ", 5: "dK"}
    for bh in [int(x) for x in args.bh.split(",")]:
        ops.enc_set_option(ctx, ops.OPT_ATTN_BH, bh)
        for w in [int(x) for x in args.which.split(",")]:
            ts = []
            for _ in range(args.reps):
                flush.fill_(1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                ops.enc_attn_gemm(ctx, w, B, H, J, P, big, small, out)
                e1.record(st)
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1) * 1e3)
            med = statistics.median(ts)
            byts = big.numel() * 2 + 2 * small.numel() * 2
            print(f"bh={bh} {names[w]:3s} median {med:7.2f} us  min {min(ts):7.2f}  "
                  f"{byts / med / 1e3:6.0f} GB/s")


if __name__ == "__main__":
    main()
