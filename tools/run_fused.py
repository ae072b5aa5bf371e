#!/usr/bin/env python
"""Time (or, under ncu, just launch) the fused score kernels at config L
(B=8, H=16, J=K=512, P=64, bf16, p=0.1): enc_attn_fwd_fused and enc_attn_bwd_fused,
L2 flushed before every launch, CUDA events on the launching stream, median of --reps."""
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
    ap.add_argument("--mask", action="store_true")
    ap.add_argument("--p", type=float, default=0.1)
    args = ap.parse_args()
    import torch
    from paper_2007_00072_b200 import ops
    B, H, J, P = args.B, 16, 512, 64
    dev = torch.device("cuda", 0)
    ctx = ops.Context(0)
    bf = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(0)
    Q = torch.randn((B, H, J, P), device=dev, generator=g).to(bf)
    K = torch.randn((B, H, J, P), device=dev, generator=g).to(bf)
    dC = torch.randn((B, J, H, P), device=dev, generator=g).to(bf)
    M = torch.zeros((B, J), device=dev) if args.mask else None
    Pm = torch.empty((B, H, J, J), device=dev, dtype=bf)
    A = torch.empty_like(Pm)
    dS = torch.empty_like(Pm)
    bits = torch.zeros((B, H, J, J // 32), dtype=torch.int32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()

    def fwd():
        ops.enc_attn_fwd_fused(ctx, B, H, J, P, 0.125, Q, K, M, args.p, 2007000072, 0, 0, Pm, A,
                               keep_bits=bits)

    def bwd():
        ops.enc_attn_bwd_fused(ctx, B, H, J, P, 0.125, dC, K, Pm, args.p, 2007000072, 0, 0, dS,
                               keep_bits=bits)

    for name, fn in (("attn_fwd_fused", fwd), ("attn_bwd_fused", bwd)):
        ts = []
        for _ in range(args.reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        byts = 2 * B * H * J * J * 2 + 2 * B * H * J * P * 2
        med = statistics.median(ts)
        print(f"{name:16s} median {med:7.2f} us  min {min(ts):7.2f}  {byts / med / 1e3:7.0f} GB/s")


if __name__ == "__main__":
    main()
