#!/usr/bin/env python
"""Timeline of the tcgen05 weight-contraction kernel (debug tool, not product): builds
tools/libencoder_wtrace.so with -DENC_WGEMM_TRACE (globaltimer stamps per CTA and tile:
MMA start / last MMA committed / epilogue has the accumulator / epilogue done), runs the
fused Linear1 + BAD (and Linear2-dX + BAD-bwd) at config L once after an L2 flush and prints
per-tile means: mainloop time, epilogue time, and how long each side waited for the other.
  python tools/trace_wgemm.py --build      (here: compile)
  python tools/trace_wgemm.py              (GPU box: run)"""
import argparse
import ctypes
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "tools", "libencoder_wtrace.so")
sys.path.insert(0, ROOT)


def build():
    import __graft_entry__ as g
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2007_00072_b200", "csrc", "*.cu")))
    cmd = [g.NVCC, *g.NVCC_FLAGS, "-DENC_WGEMM_TRACE", "-o", LIB, *srcs, "-lcublasLt",
           "-lcublas", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)


def report(name, tr):
    import numpy as np
    t = tr.reshape(148, 8, 4).astype(np.int64)
    valid = t[:, :, 0] > 0
    t0 = t[t > 0].min()
    print(f"{name}: span {(t[t > 0].max() - t0) / 1e3:.2f} us, tiles per CTA "
          f"{valid.sum(1).min()}..{valid.sum(1).max()}")
    mma = (t[:, :, 1] - t[:, :, 0])[valid] / 1e3
    epi = (t[:, :, 3] - t[:, :, 2])[valid] / 1e3
    lag = (t[:, :, 2] - t[:, :, 1])[valid] / 1e3
    print(f"  mean per tile: mainloop {mma.mean():.2f} us, epilogue {epi.mean():.2f} us, "
          f"commit->epilogue start {lag.mean():.2f} us")
    # MMA waiting for a free accumulator: start of tile it vs epilogue end of tile it-2
    w = []
    for c in range(148):
        for i in range(2, 8):
            if t[c, i, 0] > 0 and t[c, i - 2, 3] > 0:
                w.append((t[c, i, 0] - t[c, i - 1, 1]) / 1e3)
    if w:
        print(f"  MMA idle between tiles (start of tile i - commit of tile i-1): "
              f"mean {sum(w) / len(w):.2f} us")
    first = (t[:, 0, 0][valid[:, 0]] - t0) / 1e3
    last = (t.max(axis=(1, 2)) - t0) / 1e3
    print(f"  first tile start {first.min():.2f}..{first.max():.2f} us, CTA end "
          f"min {last.min():.2f} median {np.median(last):.2f} max {last.max():.2f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    a = ap.parse_args()
    if a.build:
        build()
        return
    os.environ["ENC_LIB_PATH"] = LIB   # the package binds to the traced build
    import torch
    from paper_2007_00072_b200 import _abi, ops
    lib = _abi.load()
    lib.enc_debug_wgemm_trace.argtypes = [ctypes.c_void_p, ctypes.c_size_t]
    ctx = ops.Context(0)
    B, J, I, U = 8, 512, 1024, 4096
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(0)
    X1 = torch.randn((B * J, I), device=dev, generator=g).to(torch.bfloat16)
    W1 = (0.03 * torch.randn((U, I), device=dev, generator=g)).to(torch.bfloat16)
    b1 = torch.zeros(U, device=dev)
    h = torch.empty((B * J, U), device=dev, dtype=torch.bfloat16)
    A1 = torch.empty_like(h)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    buf = (ctypes.c_ulonglong * (148 * 8 * 4))()
    for rep in range(2):
        lib.enc_debug_wgemm_trace_clear()
        flush.fill_(1)
        torch.cuda.synchronize()
        ops.enc_linear1_bad_fwd(ctx, B, J, I, U, X1, W1, b1, 0, 0.1, 7, 2, 0, h, A1)
        torch.cuda.synchronize()
        lib.enc_debug_wgemm_trace(buf, ctypes.sizeof(buf))
    import numpy as np
    report("Linear1 + BAD", np.frombuffer(buf, dtype=np.uint64))


if __name__ == "__main__":
    main()
