#!/usr/bin/env python
"""Phase timeline of the fused score kernels at config L (debug tool, not product).

Builds tools/libencoder_trace.so with -DENC_FUSED_TRACE (globaltimer stamps at the phase
boundaries of every tile, warps 0 and 31 of every CTA), runs enc_attn_fwd_fused and
enc_attn_bwd_fused once each after an L2 flush and prints the mean duration of each phase.
  python tools/trace_fused.py --build      (here: compile)
  python tools/trace_fused.py              (GPU box: run)
"""
import argparse
import ctypes
import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "tools", "libencoder_trace.so")
sys.path.insert(0, ROOT)

FWD = ["philox", "mma_wait", "pass1", "qbar", "pass2+store", "next"]
BWD = ["bits", "mma_wait", "p_wait", "pass1", "qbar", "pass2", "store+load", "next"]
FAV = ["flags", "mma_wait", "pass1", "pass2", "A_write", "av/C", "next"]


def build(extra=()):
    import __graft_entry__ as g
    srcs = sorted(glob.glob(os.path.join(ROOT, "paper_2007_00072_b200", "csrc", "*.cu")))
    cmd = [g.NVCC, *g.NVCC_FLAGS, "-DENC_FUSED_TRACE", *extra, "-o", LIB, *srcs, "-lcublasLt", "-lcublas",
           "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    subprocess.run(cmd, check=True)


def report(name, tr, labels, ntiles_cta):
    import numpy as np
    t = tr.reshape(148, 2, 8, 8).astype(np.int64)
    valid = t[:, :, :, 0] > 0
    t0 = t[:, :, :, 0][valid].min()
    tend = t[t > 0].max()
    print(f"{name}: kernel span (first tile start .. last stamp) {(tend - t0) / 1e3:.2f} us")
    ne = len(labels)
    for w, wn in ((0, "warp0"), (1, "warp31")):
        sums = np.zeros(ne)
        cnt = np.zeros(ne)
        for c in range(148):
            for it in range(ntiles_cta):
                row = t[c, w, it]
                if row[0] == 0:
                    continue
                nxt = t[c, w, it + 1, 0] if it + 1 < 8 and t[c, w, it + 1, 0] > 0 else 0
                stamps = list(row[:ne]) + [nxt]
                for e in range(ne):
                    a, b = stamps[e], stamps[e + 1]
                    if a > 0 and b > 0:
                        sums[e] += (b - a)
                        cnt[e] += 1
        line = "  ".join(f"{labels[e]} {sums[e] / max(cnt[e], 1) / 1e3:6.2f}" for e in range(ne))
        print(f"  {wn} mean us per tile: {line}")
    if ne == 7:   # the fused score + A.V kernel: warp 31 stamps 7 (C ready) between 5 and 6
        r = t[:, 1, :ntiles_cta]
        ok = (r[..., 5] > 0) & (r[..., 7] > 0) & (r[..., 6] > 0)
        if ok.any():
            a = ((r[..., 7] - r[..., 5])[ok]).mean() / 1e3
            b = ((r[..., 6] - r[..., 7])[ok]).mean() / 1e3
            print(f"  warp31: A written -> C ready {a:6.2f} us  C read-out + store {b:6.2f} us")
    starts = np.sort(t[:, 0, 0, 0][t[:, 0, 0, 0] > 0] - t0) / 1e3
    print(f"  CTA first-tile start spread: {starts[0]:.2f} .. {starts[-1]:.2f} us")
    ends = []
    for c in range(148):
        row = t[c, 0]
        if not (row > 0).any():
            continue
        ends.append((row[row > 0].max() - t0) / 1e3)
    ends = np.sort(np.array(ends))
    print(f"  CTA last-stamp: min {ends[0]:.2f} median {np.median(ends):.2f} max {ends[-1]:.2f} us")


def run():
    os.environ["ENC_LIB_PATH"] = LIB
    import numpy as np
    import torch
    from paper_2007_00072_b200 import _abi, ops
    lib = _abi.load()
    B, H, J, P = 8, 16, 512, 64
    dev = torch.device("cuda", 0)
    ctx = ops.Context(0)
    bf = torch.bfloat16
    g = torch.Generator(device=dev).manual_seed(0)
    Q = torch.randn((B, H, J, P), device=dev, generator=g).to(bf)
    K = torch.randn((B, H, J, P), device=dev, generator=g).to(bf)
    dC = torch.randn((B, J, H, P), device=dev, generator=g).to(bf)
    Pm = torch.empty((B, H, J, J), device=dev, dtype=bf)
    dS = torch.empty_like(Pm)
    bits = torch.zeros((B, H, J, J // 32), dtype=torch.int32, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    buf = np.zeros(148 * 2 * 8 * 8, dtype=np.uint64)

    def fwd():
        ops.enc_attn_fwd_fused(ctx, B, H, J, P, 0.125, Q, K, None, 0.1, 2007000072, 0, 0, Pm, None,
                               keep_bits=bits)

    V = torch.randn((B, H, J, P), device=dev, generator=g).to(bf)
    Cm = torch.empty((B, J, H, P), device=dev, dtype=bf)
    Clo = torch.empty_like(Cm)

    def fav():
        ops.enc_attn_fwd_fused_av(ctx, B, H, J, P, 0.125, Q, K, V, None, 0.1, 2007000072, 0, 0,
                                  Pm, bits, Cm, Clo)

    def bwd():
        ops.enc_attn_bwd_fused(ctx, B, H, J, P, 0.125, dC, K, Pm, 0.1, 2007000072, 0, 0, dS,
                               keep_bits=bits)

    for name, fn, labels in (("fwd", fwd, FWD), ("fwd_av", fav, FAV), ("bwd", bwd, BWD)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        for rep in range(2):
            lib.enc_debug_fused_trace_clear()
            flush.fill_(rep)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            lib.enc_debug_fused_trace(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
            print(f"{name} rep {rep}: event time {e0.elapsed_time(e1) * 1e3:.2f} us")
        report(name, buf, labels, 8)
        if os.path.isdir(os.path.join(ROOT, "gpurun_out")):
            np.save(os.path.join(ROOT, "gpurun_out", f"trace_{name}.npy"), buf)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--build", action="store_true")
    a = ap.parse_args()
    build() if a.build else run()
