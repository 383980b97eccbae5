"""Time 1D plans of several sizes (forward), per-pass HBM throughput."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0103001_b200 as b  # noqa: E402

for m in [int(a) for a in (sys.argv[1:] or ["24", "26", "27", "28", "29", "30"])]:
    n = 1 << m
    batch = max(1, (1 << 28) // n)
    x = torch.randn(batch, n, dtype=torch.complex64, device="cuda")
    y = torch.empty_like(x)
    p = b.Plan((n,), batch=batch, stream=torch.cuda.current_stream())
    for _ in range(2):
        p.forward(x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        p.forward(x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    passes = p.last_launch_count()
    gbs = 16.0 * n * batch * passes / (ms / 1e3) / 1e9
    print(f"m={m} batch={batch} passes={passes} {ms:.3f} ms  {gbs:.0f} GB/s per-pass HBM", flush=True)
    p.destroy()
    del x, y
    torch.cuda.empty_cache()
