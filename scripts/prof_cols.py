"""One 2D Gaussian pipeline (N x N) for ncu captures of the column kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

N = int(os.environ.get("N2D", "8192"))
x = torch.from_numpy(fixtures.complex_input(N * N, 0, seed=4).reshape(N, N)).cuda()
o = torch.empty_like(x)
p = b.Plan((N, N))
p.filter_pipeline(x, o, b.FILTER_GAUSS, 0.1)
torch.cuda.synchronize()
print("ok")
