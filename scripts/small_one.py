"""cfg2-small (f32 dottf 2^16) through the single-cluster path, a few launches (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
x = tfb.philox_fill("normal", 1 << 16, seed=1, stream=0, dtype=torch.float32)
y = tfb.philox_fill("normal", 1 << 16, seed=1, stream=1, dtype=torch.float32)
for _ in range(3):
    r = tfb.reduce(tfb.Method.TWOFOLD_FAST, x, y)
torch.cuda.synchronize()
print(_lib.lib().tf_last_launch().decode(), r.tolist())
