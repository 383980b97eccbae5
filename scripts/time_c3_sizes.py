"""C3-style real pipeline (two real-pair row passes) at several sizes, cold
and warm L2: is the ~20 us per pass a latency floor or a throughput bound?"""
import os
import sys
import statistics

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

s = torch.cuda.Stream()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
junk = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for N, M in [(256, 2048), (512, 2048), (1024, 2048), (2048, 2048), (2048, 1024), (2048, 512)]:
    x = torch.from_numpy(fixtures.sky_image(N, M, seed=3, nsrc=50)).cuda()
    o = torch.empty((N, M), dtype=torch.complex64, device="cuda")
    p = b.Plan((N, M), flags=b.IN_REAL_F32, stream=s)
    for _ in range(3):
        p.filter_pipeline(x, o, b.FILTER_GAUSS, 0.1)
    res = {}
    for mode in ("cold_w", "cold_rw", "warm"):
        evs = []
        with torch.cuda.stream(s):
            for _ in range(30):
                if mode != "warm":
                    flush.zero_()
                    if mode == "cold_rw":
                        junk.sum()  # evict the flush's dirty lines (write-back outside the timed region)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(s)
                p.filter_pipeline(x, o, b.FILTER_GAUSS, 0.1)
                e1.record(s)
                evs.append((e0, e1))
        torch.cuda.synchronize()
        res[mode] = statistics.median(a.elapsed_time(c) for a, c in evs) * 1e3
    print(f"{N}x{M}: cold(write flush) {res['cold_w']:.1f} us, cold(write+read) {res['cold_rw']:.1f} us, "
          f"warm {res['warm']:.1f} us", flush=True)
    p.destroy()
