#!/usr/bin/env python
"""Median CUDA-event time of one fused score + A.V launch and one fused BSB-bwd (row term
from C) launch at config L (B=8, H=16, J=512, P=64, dropout 0.1), L2 flushed before each
launch.  ENC_LIB_PATH selects the library build, so two builds can be compared on one box:
  python tools/time_fused_av.py [reps]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2007_00072_b200 import ops
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
    B, H, J, P = 8, 16, 512, 64
    dev = torch.device("cuda", 0)
    ctx = ops.Context(0)
    bf = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(0)
    Q, K, V = (torch.randn((B, H, J, P), device=dev, generator=g).to(bf) for _ in range(3))
    Pm = torch.empty((B, H, J, J), device=dev, dtype=bf)
    bits = torch.zeros((B, H, J, J // 32), dtype=torch.int32, device=dev)
    Cm = torch.empty((B, J, H, P), device=dev, dtype=bf)
    Clo = torch.empty_like(Cm)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    dC = torch.randn((B, J, H, P), device=dev, generator=g).to(bf)
    dS = torch.empty_like(Pm)

    def fwd():
        ops.enc_attn_fwd_fused_av(ctx, B, H, J, P, 0.125, Q, K, V, None, 0.1, 2007000072, 0, 0,
                                  Pm, bits, Cm, Clo)

    def bwd():
        ops.enc_attn_bwd_fused_dc(ctx, B, H, J, P, 0.125, dC, V, Pm, Cm, Clo, 0.1, 2007000072,
                                  0, 0, dS, keep_bits=bits)

    lib = os.path.basename(os.environ.get("ENC_LIB_PATH", "libencoder.so"))
    for name, fn in (("fused A.V", fwd), ("fused BSB-bwd (C)", bwd)):
        ts = []
        for i in range(reps + 5):
            flush.fill_(i & 255)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(e0.elapsed_time(e1) * 1e3)
        ts.sort()
        print(f"{lib}: {name} median {statistics.median(ts):.2f} us  p10 {ts[len(ts) // 10]:.2f}"
              f"  p90 {ts[9 * len(ts) // 10]:.2f}")


if __name__ == "__main__":
    main()
