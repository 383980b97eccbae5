"""Small invocations of every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per call; T4)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402


def run1d(n, batch, prec=b.C64, virt=0):
    dt = torch.complex64 if prec == b.C64 else torch.complex128
    x = torch.randn(batch, n, dtype=dt, device="cuda")
    y = torch.empty_like(x)
    p = b.Plan((n,), batch=batch, precision=prec)
    if virt:
        p.set_virtual_ranks(virt)
    p.forward(x, y)
    p.inverse(y, x)
    torch.cuda.synchronize()
    p.destroy()


def run2d(N, M, real=False, virt=0, filt=b.FILTER_GAUSS, param=0.1):
    p = b.Plan((N, M), flags=b.IN_REAL_F32 if real else 0)
    if virt:
        p.set_virtual_ranks(virt)
    x = torch.rand(N, M, device="cuda") if real else torch.randn(N, M, dtype=torch.complex64, device="cuda")
    o = torch.empty(N, M, dtype=torch.complex64, device="cuda")
    p.filter_pipeline(x, o, filt, param)
    if not real:
        p.forward(x, o)
        p.inverse(o, x)
    torch.cuda.synchronize()
    p.destroy()


for n in (8, 256, 2048, 8192):
    run1d(n, 3)                      # k_rows / k_rows_tma
run1d(1024, 2, prec=b.C128)
run1d(65536, 3)                      # k_cluster2 (default variant)
run1d(1 << 17, 2)                    # k_pass, 2 passes
run1d(1 << 21, 1)                    # k_pass, 3 passes
run1d(1 << 16, 1, virt=4)            # distributed four-step (transpose, twiddle)
run2d(256, 256, real=True)           # separable: k_rows_tma FILT + k_cols_pipe
run2d(128, 64, filt=b.FILTER_IDEAL_LITERAL, param=30.0)  # literal 3-pass
run2d(8192, 16)                      # k_cols R=8192
run2d(256, 512, virt=4)              # slab schedule, blocked k_rows
print("sanitize_small ok")
