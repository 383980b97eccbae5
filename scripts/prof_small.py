"""Small invocation of the hot kernels for ncu captures (one launch each)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda:0")
if which in ("all", "c2"):
    batch = int(os.environ.get("C2_BATCH", "4096"))
    x = torch.from_numpy(fixtures.complex_input(batch * 65536, 1, seed=2).reshape(batch, 65536)).to(dev)
    y = torch.empty_like(x)
    p = b.Plan((65536,), batch=batch)
    p.forward(x, y)
    torch.cuda.synchronize()
    p.forward(x, y)
    torch.cuda.synchronize()
if which in ("all", "r32k"):  # 32768-point rows (k_ab_st<32768>), 32768 rows
    x = torch.from_numpy(fixtures.complex_input(32768 * 32768, 1, seed=7).reshape(32768, 32768)).to(dev)
    y = torch.empty_like(x)
    p = b.Plan((32768,), batch=32768)
    p.forward(x, y)
    torch.cuda.synchronize()
    p.forward(x, y)
    torch.cuda.synchronize()
    del x, y
if which in ("all", "c3"):
    img = torch.from_numpy(fixtures.sky_image(2048, 2048, seed=3)).to(dev)
    out = torch.empty((2048, 2048), dtype=torch.complex64, device=dev)
    p = b.Plan((2048, 2048), flags=b.IN_REAL_F32)
    p.filter_pipeline(img, out, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    p.filter_pipeline(img, out, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
if which in ("all", "c4"):
    x = torch.from_numpy(fixtures.complex_input(8192 * 8192, 0, seed=4).reshape(8192, 8192)).to(dev)
    out = torch.empty_like(x)
    p = b.Plan((8192, 8192))
    p.filter_pipeline(x, out, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    p.filter_pipeline(x, out, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
if which in ("all", "c5"):
    n = 1 << 30
    x = torch.from_numpy(fixtures.complex_input(n, 1, seed=5)).to(dev)
    p = b.Plan((n,))
    y = torch.empty_like(x)
    p.forward(x, y)
    torch.cuda.synchronize()
    p.forward(x, y)
    torch.cuda.synchronize()
print("ok")
