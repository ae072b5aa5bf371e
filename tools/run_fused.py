#!/usr/bin/env python
"""Time (or, under ncu, just launch) the fused score kernels on their own: config L
(B=8, H=16, J=K=512) or Bb (--config Bb: B=96, H=12, J=K=128), P=64, bf16, p=0.1.
Variants: fwd (P + keep words, the layer's default launch: A not stored), fwd+A, fwd with
precomputed keep words (keep_pre) and the keep-word kernel alone, bwd.  L2 flushed before
every launch, CUDA events on the launching stream, median of --reps."""
import argparse
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--config", default="L", choices=["L", "Bb"])
    ap.add_argument("--mask", action="store_true")
    ap.add_argument("--p", type=float, default=0.1)
    ap.add_argument("--only", default="", help="comma list of variants to run")
    args = ap.parse_args()
    import torch
    from paper_2007_00072_b200 import ops
    B, H, J = (8, 16, 512) if args.config == "L" else (96, 12, 128)
    P = 64
    dev = torch.device("cuda", 0)
    ctx = ops.Context(0)
    bf = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(0)
    Q = torch.randn((B, H, J, P), device=dev, generator=g).to(bf)
    K = torch.randn((B, H, J, P), device=dev, generator=g).to(bf)
    dC = torch.randn((B, J, H, P), device=dev, generator=g).to(bf)
    Cm = torch.randn((B, J, H, P), device=dev, generator=g).to(bf)
    M = torch.zeros((B, J), device=dev) if args.mask else None
    Pm = torch.empty((B, H, J, J), device=dev, dtype=bf)
    A = torch.empty_like(Pm)
    dS = torch.empty_like(Pm)
    bits = torch.zeros((B, H, J, J // 32), dtype=torch.int32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()
    seed = 2007000072
    s_bytes, x_bytes, k_bytes = B * H * J * J * 2, B * H * J * P * 2, B * H * J * J // 8

    variants = {
        "fwd": (lambda: ops.enc_attn_fwd_fused(ctx, B, H, J, P, 0.125, Q, K, M, args.p, seed, 0,
                                               0, Pm, None, keep_bits=bits),
                2 * x_bytes + s_bytes + k_bytes),
        "fwd+A": (lambda: ops.enc_attn_fwd_fused(ctx, B, H, J, P, 0.125, Q, K, M, args.p, seed,
                                                 0, 0, Pm, A, keep_bits=bits),
                  2 * x_bytes + 2 * s_bytes + k_bytes),
        "keep_bits": (lambda: ops.enc_attn_keep_bits(ctx, B, H, J, J, args.p, seed, 0, 0, bits),
                      k_bytes),
        "fwd_pre": (lambda: ops.enc_attn_fwd_fused_bits(ctx, B, H, J, P, 0.125, Q, K, M, args.p,
                                                        seed, 0, 0, Pm, None, bits),
                    2 * x_bytes + s_bytes + k_bytes),
        "bwd": (lambda: ops.enc_attn_bwd_fused(ctx, B, H, J, P, 0.125, dC, K, Pm, args.p, seed, 0,
                                               0, dS, keep_bits=bits),
                2 * x_bytes + 2 * s_bytes + k_bytes),
        "fwd_av": (lambda: ops.enc_attn_fwd_fused_av(ctx, B, H, J, P, 0.125, Q, K, K, M, args.p,
                                                     seed, 0, 0, Pm, bits, Cm, Cm),
                   3 * x_bytes + s_bytes + k_bytes + 2 * x_bytes),
        "bwd_dc": (lambda: ops.enc_attn_bwd_fused_dc(ctx, B, H, J, P, 0.125, dC, K, Pm, Cm, Cm, args.p,
                                                     seed, 0, 0, dS, keep_bits=bits),
                   4 * x_bytes + 2 * s_bytes + k_bytes),
    }
    only = [v for v in args.only.split(",") if v] or list(variants)
    for name in only:
        fn, byts = variants[name]
        fn()   # bits for the backward variants (and warm-up)
        torch.cuda.synchronize()
        # the launch replayed from a CUDA graph: no host-side tensor-map encoding inside
        # the events
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        ts = []
        for _ in range(args.reps):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            gr.replay()
            e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        med = statistics.median(ts)
        print(f"{args.config} {name:10s} median {med:7.2f} us  min {min(ts):7.2f}  "
              f"{byts / med / 1e3:7.0f} GB/s (algorithmic {byts / 1e6:.1f} MB)")


if __name__ == "__main__":
    main()
