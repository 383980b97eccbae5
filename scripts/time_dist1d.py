"""C5 shape (n = 2^30 forward) through the distributed four-step on P virtual
ranks: fused distributed transposes vs pack -> all-to-all -> unpack
(B200FFT_DIST_EXCHANGE=1).  All ranks' work serialised on one GPU."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 30
n = 1 << m
x = torch.from_numpy(fixtures.complex_input(n, 1, seed=5)).cuda()
y = torch.empty_like(x)
s = torch.cuda.current_stream()
for P in (2, 8):
    for ex in ("0", "1"):
        os.environ["B200FFT_DIST_EXCHANGE"] = ex
        p = b.Plan((n,), batch=1)
        p.set_virtual_ranks(P)
        p.set_stream(s)
        for _ in range(2):
            p.forward(x, y)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(s)
        for _ in range(3):
            p.forward(x, y)
        ev[1].record(s)
        torch.cuda.synchronize()
        ms = ev[0].elapsed_time(ev[1]) / 3
        print(f"2^{m} P={P} {'exchange' if ex == '1' else 'fused'}: {ms:.3f} ms  launches {p.last_launch_count()}",
              flush=True)
        p.destroy()
        torch.cuda.empty_cache()
