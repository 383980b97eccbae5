"""C4 shape (8192^2 Gaussian pipeline) through the slab schedule on P virtual
ranks: fused peer-store / peer-load row passes vs the all-to-all schedule
(B200FFT_DIST_EXCHANGE=1).  Work of all ranks serialised on one GPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

N = 8192
x = torch.from_numpy(fixtures.complex_input(N * N, 1, seed=4).reshape(N, N)).cuda()
y = torch.empty_like(x)
s = torch.cuda.current_stream()
for P in (1, 2, 4, 8):
    for ex in ("0", "1"):
        if P == 1 and ex == "1":
            continue
        os.environ["B200FFT_DIST_EXCHANGE"] = ex
        p = b.Plan((N, N))
        if P > 1:
            p.set_virtual_ranks(P)
        p.set_stream(s)
        for _ in range(3):
            p.filter_pipeline(x, y, b.FILTER_GAUSS, 0.1)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(s)
        for _ in range(5):
            p.filter_pipeline(x, y, b.FILTER_GAUSS, 0.1)
        ev[1].record(s)
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 5
        print(f"P={P} {'exchange' if ex == '1' else 'fused'}: {ms:.3f} ms  launches {p.last_launch_count()}", flush=True)
        p.destroy()
