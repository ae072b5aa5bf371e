"""Launch torch copies of the fused-op traffic sizes (for an ncu speed-of-light reference)."""
import torch
for mb in (16.8, 25.2, 33.6, 50.3, 100.7):
    n = int(mb * 1e6 / 2)
    a = torch.randn(n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty_like(a)
    b.copy_(a)
torch.cuda.synchronize()
