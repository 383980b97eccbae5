"""Microbenchmark: L2-resident copy bandwidth vs HBM copy bandwidth (torch copy_)."""
import torch

for mb in (8, 16, 32, 48, 64, 96, 256, 2048):
    n = mb * (1 << 20) // 4
    a = torch.randn(n, device="cuda")
    b = torch.empty_like(a)
    for _ in range(5):
        b.copy_(a)
    torch.cuda.synchronize()
    reps = 200 if mb <= 96 else 20
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        b.copy_(a)
    e.record()
    torch.cuda.synchronize()
    t = s.elapsed_time(e) / reps
    print(f"{mb:5d} MiB copy: {t * 1e3:8.2f} us  {2 * mb * (1 << 20) / (t / 1e3) / 1e9:8.0f} GB/s (read+write)")
