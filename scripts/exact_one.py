"""One exact-sum launch on 2^26 f64 (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402

torch.cuda.set_device(0)
x = tfb.philox_fill("uniform_sym", 1 << 26, seed=1)
for _ in range(3):
    r = tfb.exact_sum(x)
torch.cuda.synchronize()
print(r.hi)
