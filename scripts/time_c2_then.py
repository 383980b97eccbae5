"""C2 (k_ab_st) then C4 / C5 in the same process: does the C2 ring's L2
persistence slow the following workloads?  Prints C2, C4 and C5 times."""
import os
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(here))
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

n, batch = 65536, 4096
x = torch.from_numpy(fixtures.complex_input(batch * n, 1, seed=2).reshape(batch, n)).cuda()
y = torch.empty_like(x)
st = torch.cuda.Stream()
p = b.Plan((n,), batch=batch, stream=st)
for _ in range(3):
    p.forward(x, y)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(st)
for _ in range(10):
    p.forward(x, y)
e.record(st)
torch.cuda.synchronize()
print(f"C2 fwd {s.elapsed_time(e) / 10:.4f} ms", flush=True)
p.destroy()
del x, y
torch.cuda.empty_cache()
sys.argv = [sys.argv[0]]
exec(open(os.path.join(here, "time_c4c5.py")).read())
