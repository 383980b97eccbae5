"""One C5 forward transform (N = 2^30 complex64) for ncu captures."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

m = int(os.environ.get("C5_LOG2", "30"))
n = 1 << m
x = np.empty(n, np.complex64)
fixtures.complex_input(n, fixtures.NORMAL, seed=5, out=x)
xd = torch.from_numpy(x).cuda()
yd = torch.empty_like(xd)
p = b.Plan((n,), batch=1)
p.forward(xd, yd)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
p.forward(xd, yd)
e.record()
torch.cuda.synchronize()
print(f"forward 2^{m}: {s.elapsed_time(e):.3f} ms")
