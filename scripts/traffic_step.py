"""One warm-up step, then ONE profiled step (cudaProfilerStart/Stop) of a
config's hot path, for `ncu --profile-from-start off` captures of every
kernel's DRAM bytes and time (scripts/gpu_traffic.sh).
usage: traffic_step.py C2|C3|C3_real|C4|C5"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

cfg = sys.argv[1]
dev = torch.device("cuda:0")
if cfg == "C2":
    x = torch.from_numpy(fixtures.complex_input(4096 * 65536, 1, seed=2).reshape(4096, 65536)).to(dev)
    y = torch.empty_like(x)
    p = b.Plan((65536,), batch=4096)
    step = lambda: p.forward(x, y)  # noqa: E731  (the roofline's dominant launch)
elif cfg in ("C3", "C3_real"):
    img = torch.from_numpy(fixtures.sky_image(2048, 2048, seed=3)).to(dev)
    real = cfg == "C3_real"
    out = torch.empty((2048, 2048), dtype=torch.float32 if real else torch.complex64, device=dev)
    p = b.Plan((2048, 2048), flags=b.IN_REAL_F32 | (b.OUT_REAL_F32 if real else 0))
    step = lambda: p.filter_pipeline(img, out, b.FILTER_GAUSS, 0.1)  # noqa: E731
elif cfg == "C4":
    x = torch.from_numpy(fixtures.complex_input(8192 * 8192, 0, seed=4).reshape(8192, 8192)).to(dev)
    out = torch.empty_like(x)
    p = b.Plan((8192, 8192))
    step = lambda: p.filter_pipeline(x, out, b.FILTER_GAUSS, 0.1)  # noqa: E731
elif cfg == "C4_real":
    img = torch.from_numpy(fixtures.sky_image(8192, 8192, seed=4, nsrc=2000)).to(dev)
    out = torch.empty_like(img)
    p = b.Plan((8192, 8192), flags=b.IN_REAL_F32 | b.OUT_REAL_F32)
    step = lambda: p.filter_pipeline(img, out, b.FILTER_GAUSS, 0.1)  # noqa: E731
elif cfg == "C5":
    n = 1 << 30
    xh = np.empty(n, np.complex64)
    fixtures.complex_input(n, 1, seed=5, out=xh)
    x = torch.from_numpy(xh).to(dev)
    del xh
    y, z = torch.empty_like(x), torch.empty_like(x)
    p = b.Plan((n,))

    def step():
        p.forward(x, y)
        p.inverse(y, z)
else:
    raise SystemExit(f"unknown config {cfg}")
step()
torch.cuda.synchronize()
torch.cuda.profiler.start()
step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok", cfg)
