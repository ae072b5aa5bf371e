"""Run one weight contraction of config L a few times eagerly (ncu target).
usage: python tools/run_wgemm.py {l1_bad|l2dx_bad|fwd|dx|dw} [M N K] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2007_00072_b200 import ops  # noqa: E402

which = sys.argv[1]
M, N, K = (int(x) for x in sys.argv[2:5]) if len(sys.argv) >= 5 else (4096, 4096, 1024)
reps = int(sys.argv[5]) if len(sys.argv) >= 6 else 3
ctx = ops.Context(0)
bf = torch.bfloat16
A = torch.randn(M, K, device="cuda", dtype=bf)
for _ in range(reps):
    if which == "l1_bad":
        W = torch.randn(N, K, device="cuda", dtype=bf) * 0.03
        h = torch.empty(M, N, device="cuda", dtype=bf)
        A1 = torch.empty_like(h)
        ops.enc_linear1_bad_fwd(ctx, M // 512, 512, K, N, A, W, torch.zeros(N, device="cuda"),
                                0, 0.1, 1, 2, 0, h, A1)
    elif which == "l2dx_bad":
        W = torch.randn(K, N, device="cuda", dtype=bf) * 0.03
        h = torch.randn(M, N, device="cuda", dtype=bf)
        dh = torch.empty_like(h)
        db = torch.empty(N, device="cuda")
        ops.enc_linear2_dx_bad_bwd(ctx, M // 512, 512, K, N, A, W, h, 0, 0.1, 1, 2, 0, dh, db)
    elif which == "fwd":
        W = torch.randn(N, K, device="cuda", dtype=bf)
        C = torch.empty(M, N, device="cuda", dtype=bf)
        ops.enc_wgemm(ctx, A, W, C, tA=False, tB=True)
    elif which == "dx":
        W = torch.randn(K, N, device="cuda", dtype=bf)
        C = torch.empty(M, N, device="cuda", dtype=bf)
        ops.enc_wgemm(ctx, A, W, C, tA=False, tB=False)
    else:
        At = torch.randn(K, M, device="cuda", dtype=bf)
        B = torch.randn(K, N, device="cuda", dtype=bf)
        C = torch.empty(M, N, device="cuda", dtype=torch.float32)
        ops.enc_wgemm(ctx, At, B, C, tA=True, tB=False)
torch.cuda.synchronize()
print("done")
