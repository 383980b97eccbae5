"""time_1d.py against a given libb200fft.so (A/B timing of two builds):
python scripts/time_1d_lib.py LIB m1 m2 ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_cs_0103001_b200 as b  # noqa: E402

b.load_library(sys.argv[1])
for m in [int(a) for a in sys.argv[2:]]:
    n = 1 << m
    batch = max(1, (1 << 28) // n) if m < 30 else 1
    x = torch.randn(batch, n, dtype=torch.complex64, device="cuda")
    y = torch.empty_like(x)
    p = b.Plan((n,), batch=batch, stream=torch.cuda.current_stream())
    for _ in range(2):
        p.forward(x, y)
        p.inverse(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        p.forward(x, y)
        p.inverse(y, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"{os.path.basename(os.path.dirname(sys.argv[1]))} m={m} fwd+inv {ms:.3f} ms", flush=True)
    p.destroy()
    del x, y
    torch.cuda.empty_cache()
