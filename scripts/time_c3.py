"""Time the C3 / C4 2D Gaussian pipelines (cold L2) with the current env knobs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402


def run(N, real, reps=20, real_out=False):
    s = torch.cuda.current_stream()
    if real:
        x = torch.from_numpy(fixtures.sky_image(N, N, seed=3)).cuda()
        p = b.Plan((N, N), flags=b.IN_REAL_F32 | (b.OUT_REAL_F32 if real_out else 0), stream=s)
    else:
        x = torch.from_numpy(fixtures.complex_input(N * N, 0, seed=4).reshape(N, N)).cuda()
        p = b.Plan((N, N), stream=s)
    o = torch.empty((N, N), dtype=torch.float32 if real_out else torch.complex64, device="cuda")
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        p.filter_pipeline(x, o, b.FILTER_GAUSS, 0.1)
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        p.filter_pipeline(x, o, b.FILTER_GAUSS, 0.1)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    med = ts[len(ts) // 2]
    alg = (16.0 if real_out else 32.0) * N * N
    print(f"N={N} real={real} real_out={real_out}: "
          f"median {med * 1e3:.1f} us  min {ts[0] * 1e3:.1f} us  hbm_frac {alg / (med / 1e3) / 1e9 / 6554.6:.3f}",
          flush=True)


if __name__ == "__main__":
    run(2048, True)
    run(2048, True, real_out=True)
    run(8192, False, reps=10)
