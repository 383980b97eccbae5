"""C1 (1024-point complex128, forward + inverse): a few reps for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

x = torch.from_numpy(fixtures.complex_input(1024, fixtures.UNIFORM, seed=1, dtype=np.complex128)).cuda()
y, z = torch.empty_like(x), torch.empty_like(x)
p = b.Plan((1024,), batch=1, precision=b.C128)
for _ in range(4):
    p.forward(x, y)
    p.inverse(y, z)
torch.cuda.synchronize()
print(float((z - x).abs().max()))
