"""Speed-of-light reference: torch copy (read N + write N bytes) at the fused-op sizes of
config L, CUDA-event timed (median of 30), with the L2 flushed before each launch either by
WRITING a 512 MB buffer (leaves ~126 MB of dirty lines to be written back during the timed
kernel) or by READING one (leaves clean lines)."""
import statistics
import torch

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
sink = torch.empty(1, dtype=torch.int64, device="cuda")
for mode in ("write-flush", "read-flush"):
    for mb in (8.4, 16.8, 33.6, 67.1, 100.7, 268.4):
        n = int(mb * 1e6 / 2)
        a = torch.randn(n, device="cuda", dtype=torch.bfloat16)
        b = torch.empty_like(a)
        ts = []
        for r in range(35):
            if mode == "write-flush":
                flush.zero_()
            else:
                torch.sum(flush.view(torch.int64), dim=0, out=sink[0])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); b.copy_(a); e1.record(); torch.cuda.synchronize()
            if r >= 5:
                ts.append(e0.elapsed_time(e1))
        t = statistics.median(ts) * 1e-3
        print(f"{mode:11s} copy {mb:6.1f} MB + {mb:6.1f} MB: {t*1e6:7.1f} us  {2*mb*1e6/t/1e9:7.0f} GB/s")
