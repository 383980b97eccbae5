"""C4 (8192^2 pipeline) and C5 (2^30 fwd+inv) at P=1: back-to-back event
timing vs per-rep synchronised timing, to cross-check bench.py."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

which = sys.argv[1:] or ["C4", "C5"]
st = torch.cuda.Stream()
for cfg in which:
    if cfg == "C4":
        N = 8192
        x = torch.from_numpy(fixtures.complex_input(N * N, 0, seed=4).reshape(N, N)).cuda()
        y = torch.empty_like(x)
        p = b.Plan((N, N), stream=st)
        step = lambda: p.filter_pipeline(x, y, b.FILTER_GAUSS, 0.1)  # noqa: E731
        reps = 20
    else:
        n = 1 << 30
        xh = np.empty(n, np.complex64)
        fixtures.complex_input(n, 1, seed=5, out=xh)
        x = torch.from_numpy(xh).cuda()
        del xh
        y, z = torch.empty_like(x), torch.empty_like(x)
        p = b.Plan((n,), stream=st)

        def step():
            p.forward(x, y)
            p.inverse(y, z)
        reps = 6
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for _ in range(reps):
        step()
    e.record(st)
    torch.cuda.synchronize()
    bb = s.elapsed_time(e) / reps
    evs = []
    for _ in range(reps):
        a, c = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        step()
        c.record(st)
        evs.append((a, c))
    torch.cuda.synchronize()
    per = [a.elapsed_time(c) for a, c in evs]
    print(f"{cfg}: back-to-back {bb:.4f} ms/step; per-rep events median {statistics.median(per):.4f} min {min(per):.4f}",
          flush=True)
    del x, y
    p.destroy()
    torch.cuda.empty_cache()
