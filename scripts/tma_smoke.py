"""Short TMA-loader smoke: results must equal the LDG loader's bit for bit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402

L = _lib.lib()
torch.cuda.set_device(0)
for dt in (torch.float32, torch.float64):
    for n in (5000, 100_003, 1 << 20, (1 << 22) + 9):
        x = tfb.philox_fill("uniform_sym", n, seed=1, stream=0, dtype=dt)
        y = tfb.philox_fill("uniform_sym", n, seed=1, stream=1, dtype=dt)
        for meth in (tfb.Method.TWOFOLD_FAST, tfb.Method.KAHAN):
            L.tf_set_loader(0)
            a = tfb.reduce(meth, x, y).cpu()
            for ld in (1, 2):
                L.tf_set_loader(ld)
                b = tfb.reduce(meth, x, y).cpu()
                torch.cuda.synchronize()
                assert torch.equal(a, b), (dt, n, meth, ld, a, b)
print("tma smoke ok")
