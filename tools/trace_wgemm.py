import ctypes, sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2007_00072_b200 import ops, _abi
lib = _abi.load()
ctx = ops.Context(0)
M, N, K = [int(x) for x in sys.argv[1:4]]
bf = torch.bfloat16
A = torch.randn(M, K, device="cuda", dtype=bf); W = torch.randn(N, K, device="cuda", dtype=bf); C = torch.empty(M, N, device="cuda", dtype=bf)
for _ in range(3):
    ops.enc_wgemm(ctx, A, W, C, tA=False, tB=True)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (256 * 16))()
lib.enc_debug_wgemm_trace(buf)
t = np.array(buf, dtype=np.int64).reshape(256, 16)[:148]
t0 = t[:, 15].min()
rel = lambda x: (x - t0) / 1000.0
print("start spread us:", rel(t[:, 15]).min(), rel(t[:, 15]).max())
for cta in [0, 1, 2, 3, 50, 51, 100, 146, 147]:
    r = t[cta]
    print(cta, "start %.2f" % rel(r[15]), " ".join("%d:%.2f" % (i, rel(r[i])) for i in range(8) if r[i] > 0), "waitdone %.2f" % (rel(r[14]) if r[14] > 0 else -1))
