"""Time the C2 kernel (4096 x 65536 complex64, forward + inverse) for the
kernel named by B200FFT_C2, with a parity spot
check of 64 rows against the oracle.  Usage: python scripts/time_c2.py [reps]"""
import os
import sys
import statistics

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fixtures  # noqa: E402
import oracle  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
n, batch = 65536, 4096
x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=2).reshape(batch, n)
st = torch.cuda.Stream()
p = b.Plan((n,), batch=batch, stream=st)
xd = torch.from_numpy(x).cuda()
yd, zd = torch.empty_like(xd), torch.empty_like(xd)
for _ in range(3):
    p.forward(xd, yd)
    p.inverse(yd, zd)
torch.cuda.synchronize()
tf, ti = [], []
for _ in range(reps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(st)
    p.forward(xd, yd)
    e[1].record(st)
    p.inverse(yd, zd)
    e[2].record(st)
    torch.cuda.synchronize()
    tf.append(e[0].elapsed_time(e[1]))
    ti.append(e[1].elapsed_time(e[2]))
rows = np.arange(0, batch, 64)
err = oracle.rel_l2(yd[torch.from_numpy(rows).cuda()].cpu().numpy(), oracle.fft_batch(x[rows]))
rt = float(torch.linalg.vector_norm(zd - xd) / torch.linalg.vector_norm(xd))
gbs = 16.0 * n * batch / (statistics.median(tf) / 1e3) / 1e9
print(f"C2 kernel={os.environ.get('B200FFT_C2', 'default')}: fwd med {statistics.median(tf):.4f} min {min(tf):.4f} ms, "
      f"inv med {statistics.median(ti):.4f} ms, {gbs:.0f} GB/s ({gbs / 6550.4:.3f}), fwd err {err:.2e}, rt {rt:.2e}",
      flush=True)
