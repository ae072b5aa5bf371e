"""Speed-of-light reference: torch copy (read N + write N bytes) at the fused-op sizes of
config L, L2 flushed before each launch, CUDA-event timed (median of 30)."""
import statistics
import torch

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
for mb in (8.4, 16.8, 25.2, 33.6, 67.1, 100.7, 268.4):
    n = int(mb * 1e6 / 2)
    a = torch.randn(n, device="cuda", dtype=torch.bfloat16)
    b = torch.empty_like(a)
    ts = []
    for r in range(35):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
        if r >= 5:
            ts.append(e0.elapsed_time(e1))
    t = statistics.median(ts) * 1e-3
    print(f"copy read {mb:6.1f} MB + write {mb:6.1f} MB: {t*1e6:7.1f} us  {2*mb*1e6/t/1e9:7.0f} GB/s")
