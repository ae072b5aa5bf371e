"""Launch torch bf16 copies moving the algorithmic byte volumes of the fused operators at
config L (read N + write N bytes), for an ncu speed-of-light reference:
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:copy python tools/ncu_copy_ref.py
(ncu flushes the caches before every kernel, like the fused-kernel captures)."""
import torch

# total bytes (read + write) of: BDRLN fwd/bwd 33.6 MB, BAD fwd 67.1 MB, BAD bwd 100.7 MB,
# attention fused fwd/bwd 155 MB, attention stream 75.5 MB
for total_mb in (33.6, 67.1, 75.5, 100.7, 155.2):
    n = int(total_mb / 2 * 1e6 / 2)
    a = torch.randn(n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty_like(a)
    for _ in range(3):
        torch.mul(a, 1.0, out=b)   # an element-wise kernel (copy_ would be a DMA memcpy)
torch.cuda.synchronize()
