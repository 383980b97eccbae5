"""e2e (fft_execute_host on pinned host buffers) of C2: forward + inverse per
step, host wall clock; with B200FFT_HOST_CHUNK_MB from the environment."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

n, batch = 65536, 4096
xh = torch.from_numpy(fixtures.complex_input(batch * n, 1, seed=2).reshape(batch, n)).pin_memory()
oh, bh = torch.empty_like(xh).pin_memory(), torch.empty_like(xh).pin_memory()
p = b.Plan((n,), batch=batch)
p.execute_host(+1, xh, oh)
t0 = time.perf_counter()
for _ in range(3):
    p.execute_host(+1, xh, oh)
    p.execute_host(-1, oh, bh)
dt = (time.perf_counter() - t0) / 3
err = float(torch.linalg.vector_norm(bh - xh) / torch.linalg.vector_norm(xh))
print(f"e2e chunk={os.environ.get('B200FFT_HOST_CHUNK_MB', '64')} MB: {dt * 1e3:.1f} ms/step, "
      f"{2 * 5 * n * 16 * batch / dt / 1e9:.1f} GFLOP/s, {2 * 2 * 8 * n * batch / dt / 1e9:.1f} GB/s PCIe, err {err:.1e}",
      flush=True)
