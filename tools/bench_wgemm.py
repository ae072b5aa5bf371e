"""Time the hand-written tcgen05 weight contractions (enc_wgemm / the fused FFN kernels)
against cuBLAS (torch.matmul, bf16, fp32 accumulate) on the layer's shapes at configs L and
Bb.  Each contraction is replayed 20x inside one CUDA graph (no launch gaps), CUDA events
around the replay, median of 5 replays; TFLOP/s = 2MNK / time.

usage: python tools/bench_wgemm.py [--config L|Bb] [--json out.json]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def graph_time(fn, reps=20, trials=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    ts = []
    for _ in range(trials):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / reps)
    ts.sort()
    return ts[len(ts) // 2]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="L")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    from paper_2007_00072_b200 import ops
    ctx = ops.Context(0)
    ctx1 = ops.Context(0)   # single-CTA tiles, for comparison
    ops.enc_set_option(ctx1, ops.OPT_GEMM_PAIR, 0)
    BJ, I, U = (4096, 1024, 4096) if a.config == "L" else (12288, 768, 3072)
    bf = torch.bfloat16
    dev = "cuda"
    torch.manual_seed(0)
    rows = []
    # (name, M, N, K, form): fwd = X W^T, dx = dY W, dw = dY^T X (fp32 out)
    shapes = [("qkv", BJ, 3 * I, I, "fwd"), ("out", BJ, I, I, "fwd"), ("l1", BJ, U, I, "fwd"),
              ("l2", BJ, I, U, "fwd"), ("l2_dx", BJ, U, I, "dx"), ("l1_dx", BJ, I, U, "dx"),
              ("out_dx", BJ, I, I, "dx"), ("qkv_dx", BJ, I, 3 * I, "dx"),
              ("l2_dw", I, U, BJ, "dw"), ("l1_dw", U, I, BJ, "dw"), ("out_dw", I, I, BJ, "dw"),
              ("qkv_dw", 3 * I, I, BJ, "dw")]
    for name, M, N, K, form in shapes:
        if form == "fwd":
            A = torch.randn(M, K, device=dev, dtype=bf)
            B = torch.randn(N, K, device=dev, dtype=bf) * 0.02
            C = torch.empty(M, N, device=dev, dtype=bf)
            mine = lambda: ops.enc_wgemm(ctx, A, B, C, tA=False, tB=True)  # noqa: E731
            ref = lambda: torch.matmul(A, B.t(), out=C)  # noqa: E731
        elif form == "dx":
            A = torch.randn(M, K, device=dev, dtype=bf)
            B = torch.randn(K, N, device=dev, dtype=bf) * 0.02
            C = torch.empty(M, N, device=dev, dtype=bf)
            mine = lambda: ops.enc_wgemm(ctx, A, B, C, tA=False, tB=False)  # noqa: E731
            ref = lambda: torch.matmul(A, B, out=C)  # noqa: E731
        else:
            A = torch.randn(K, M, device=dev, dtype=bf)
            B = torch.randn(K, N, device=dev, dtype=bf)
            C = torch.empty(M, N, device=dev, dtype=torch.float32)
            Cb = torch.empty(M, N, device=dev, dtype=bf)
            mine = lambda: ops.enc_wgemm(ctx, A, B, C, tA=True, tB=False)  # noqa: E731
            ref = lambda: torch.matmul(A.t(), B, out=Cb)  # noqa: E731
        t_m = graph_time(mine)
        t_r = graph_time(ref)
        cs = ctx
        ctx = ctx1
        t_1 = graph_time(mine)
        ctx = cs
        fl = 2.0 * M * N * K
        rows.append({"op": name, "M": M, "N": N, "K": K, "tc_us": round(t_m, 2),
                     "cublas_us": round(t_r, 2), "tc_tflops": round(fl / t_m / 1e6, 1),
                     "cublas_tflops": round(fl / t_r / 1e6, 1)})
        print(f"{name:8s} {M:6d}x{N:5d}x{K:6d}  tc {t_m:7.2f} us {fl / t_m / 1e6:7.1f} TF/s   "
              f"cublas {t_r:7.2f} us {fl / t_r / 1e6:7.1f} TF/s   ratio {t_r / t_m:.3f}   "
              f"single-CTA {t_1:7.2f} us",
              flush=True)
    # fused FFN kernels against their unfused cuBLAS + element-wise baseline is timed by
    # the layer bench; here: the fused kernels alone
    Bq, J = (8, 512) if a.config == "L" else (96, 128)
    X1 = torch.randn(BJ, I, device=dev, dtype=bf)
    W1 = torch.randn(U, I, device=dev, dtype=bf) * 0.02
    b1 = torch.zeros(U, device=dev)
    h = torch.empty(BJ, U, device=dev, dtype=bf)
    A1 = torch.empty_like(h)
    t = graph_time(lambda: ops.enc_linear1_bad_fwd(ctx, Bq, J, I, U, X1, W1, b1, 0, 0.1, 1, 2, 0,
                                                   h, A1))
    fl = 2.0 * BJ * U * I
    rows.append({"op": "l1_bad_fused", "tc_us": round(t, 2), "tc_tflops": round(fl / t / 1e6, 1)})
    print(f"l1+BAD fused  {t:7.2f} us {fl / t / 1e6:7.1f} TF/s", flush=True)
    dY2 = torch.randn(BJ, I, device=dev, dtype=bf)
    W2 = torch.randn(I, U, device=dev, dtype=bf) * 0.02
    dh = torch.empty(BJ, U, device=dev, dtype=bf)
    db1 = torch.empty(U, device=dev)
    t = graph_time(lambda: ops.enc_linear2_dx_bad_bwd(ctx, Bq, J, I, U, dY2, W2, h, 0, 0.1, 1, 2,
                                                      0, dh, db1))
    rows.append({"op": "l2dx_badbwd_fused", "tc_us": round(t, 2),
                 "tc_tflops": round(fl / t / 1e6, 1)})
    print(f"l2dx+BAD-bwd fused  {t:7.2f} us {fl / t / 1e6:7.1f} TF/s", flush=True)
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"config": a.config, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
