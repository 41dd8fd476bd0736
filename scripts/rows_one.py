"""One row-wise launch of a given shape (for ncu): python scripts/rows_one.py ROWS COLS [f32|f64]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402

rows, cols = int(sys.argv[1]), int(sys.argv[2])
dt = torch.float64 if len(sys.argv) > 3 and sys.argv[3] == "f64" else torch.float32
torch.cuda.set_device(0)
X = torch.rand(rows, cols, dtype=dt, device="cuda")
Y = torch.rand(rows, cols, dtype=dt, device="cuda")
for _ in range(3):
    out = tfb.reduce_rows(tfb.Method.TWOFOLD_FAST, X, Y)
torch.cuda.synchronize()
print("ok", tuple(out.shape), tfb._lib.lib().tf_last_launch().decode())
