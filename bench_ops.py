#!/usr/bin/env python
"""Per-operator HBM-roofline sweep (BASELINE.json config 5, SURVEY.md 8(d) "SW"):
BSB / BSB-bwd / BDRLN / BDRLN-bwd (and BAD, AIB at the layer shape) at B=8, H=16, I=1024,
J = 128 ... 4096, bf16, through the C ABI.  Each measurement: L2 flushed (512 MB write)
before every launch, CUDA events on the launching stream, median of --reps.
Prints one JSON line per (op, J) and a table on stderr."""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--J", default="128,256,512,1024,2048,4096")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--ops", default="bsb_fwd,bsb_bwd,bdrln_fwd,bdrln_bwd,bad_fwd,bad_bwd,aib_fwd,aib_bwd")
    args = ap.parse_args()
    import torch

    import __graft_entry__
    __graft_entry__.build()
    from paper_2007_00072_b200 import ops
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = peaks["hbm_gbs"]
    dev = torch.device("cuda", 0)
    ctx = ops.Context(0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    B, H, P, I, U = 8, 16, 64, 1024, 4096
    bf = torch.bfloat16
    seed, p = 2007000072, 0.1
    wanted = args.ops.split(",")

    def timeit(fn):
        ts = []
        for r in range(args.reps + 2):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(a.elapsed_time(b))
        return statistics.median(ts) * 1e-3

    rows = []
    for J in [int(x) for x in args.J.split(",")]:
        g = torch.Generator(device=dev).manual_seed(J)
        BHJK = (B, H, J, J)
        res = {}
        if {"bsb_fwd", "bsb_bwd"} & set(wanted):
            S = torch.randn(BHJK, device=dev, dtype=bf, generator=g)
            Pm, A = torch.empty_like(S), torch.empty_like(S)
            if "bsb_fwd" in wanted:
                t = timeit(lambda: ops.enc_bsb_fwd(ctx, B, H, J, J, 0.125, S, None, p, seed, 0, 0,
                                                   Pm, A))
                res["bsb_fwd"] = (t, 3 * S.numel() * 2)
            if "bsb_bwd" in wanted:
                ops.enc_bsb_fwd(ctx, B, H, J, J, 0.125, S, None, p, seed, 0, 0, Pm, A)
                dS = torch.empty_like(S)
                t = timeit(lambda: ops.enc_bsb_bwd(ctx, B, H, J, J, 0.125, S, Pm, p, seed, 0, 0,
                                                   dS))
                res["bsb_bwd"] = (t, 3 * S.numel() * 2)
            del S, Pm, A
        if {"bdrln_fwd", "bdrln_bwd"} & set(wanted):
            Y = torch.randn((B, J, I), device=dev, dtype=bf, generator=g)
            R = torch.randn((B, J, I), device=dev, dtype=bf, generator=g)
            vec = lambda: torch.randn(I, device=dev, generator=g) * 0.1  # noqa: E731
            bias, gam, bet = vec(), vec() + 1, vec()
            out, xh = torch.empty_like(Y), torch.empty_like(Y)
            rstd = torch.empty((B, J), device=dev)
            n = B * J * I
            if "bdrln_fwd" in wanted:
                t = timeit(lambda: ops.enc_bdrln_fwd(ctx, B, J, I, Y, bias, R, gam, bet, 1e-5, p,
                                                     seed, 1, 0, out, xh, rstd))
                res["bdrln_fwd"] = (t, 4 * n * 2 + B * J * 4)
            if "bdrln_bwd" in wanted:
                ops.enc_bdrln_fwd(ctx, B, J, I, Y, bias, R, gam, bet, 1e-5, p, seed, 1, 0, out, xh,
                                  rstd)
                dz, dy = torch.empty_like(Y), torch.empty_like(Y)
                dg, db, dbi = (torch.empty(I, device=dev) for _ in range(3))
                t = timeit(lambda: ops.enc_bdrln_bwd(ctx, B, J, I, Y, xh, rstd, gam, p, seed, 1, 0,
                                                     dz, dy, dg, db, dbi))
                res["bdrln_bwd"] = (t, 4 * n * 2 + B * J * 4)
        if J == 512:   # the layer-shape-only ops
            if {"bad_fwd", "bad_bwd"} & set(wanted):
                Y1 = torch.randn((B, J, U), device=dev, dtype=bf, generator=g)
                b1 = torch.zeros(U, device=dev)
                h, A1 = torch.empty_like(Y1), torch.empty_like(Y1)
                if "bad_fwd" in wanted:
                    t = timeit(lambda: ops.enc_bad_fwd(ctx, B, J, U, Y1, b1, 0, p, seed, 2, 0, h, A1))
                    res["bad_fwd"] = (t, 3 * Y1.numel() * 2)
                if "bad_bwd" in wanted:
                    dh = torch.empty_like(Y1)
                    db1 = torch.empty(U, device=dev)
                    t = timeit(lambda: ops.enc_bad_bwd(ctx, B, J, U, Y1, h, 0, p, seed, 2, 0, dh, db1))
                    res["bad_bwd"] = (t, 3 * Y1.numel() * 2)
            if {"aib_fwd", "aib_bwd"} & set(wanted):
                qkv = torch.randn((B, J, 3 * I), device=dev, dtype=bf, generator=g)
                bq = torch.zeros(3 * I, device=dev)
                q, k, v = (torch.empty((B, H, J, P), device=dev, dtype=bf) for _ in range(3))
                if "aib_fwd" in wanted:
                    t = timeit(lambda: ops.enc_aib_fwd(ctx, B, J, H, P, qkv, bq, q, k, v))
                    res["aib_fwd"] = (t, 2 * qkv.numel() * 2)
                if "aib_bwd" in wanted:
                    dbq = torch.empty(3 * I, device=dev)
                    t = timeit(lambda: ops.enc_aib_bwd(ctx, B, J, H, P, q, k, v, qkv, dbq))
                    res["aib_bwd"] = (t, 2 * qkv.numel() * 2)
        for op, (t, nbytes) in res.items():
            gbs = nbytes / t / 1e9
            line = {"op": op, "J": J, "B": B, "H": H, "I": I, "us": t * 1e6, "bytes": nbytes,
                    "GB/s": gbs, "frac_hbm": gbs / hbm, "peak_gbs": hbm, "l2": "flushed"}
            rows.append(line)
            print(json.dumps(line), flush=True)
            print(f"{op:10s} J={J:5d} {t * 1e6:9.1f} us {gbs:8.0f} GB/s {100 * gbs / hbm:5.1f}% of {hbm}",
                  file=sys.stderr)
        torch.cuda.empty_cache()
    return rows


if __name__ == "__main__":
    main()
