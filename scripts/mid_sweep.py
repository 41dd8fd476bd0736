"""cfg2-sized sensitivity: leaf size x split x loader (full reduce, PDL tail), graph-replayed."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from tail_cost import graph_us  # noqa: E402

L = _lib.lib()
torch.cuda.set_device(0)
M = tfb.Method.TWOFOLD_FAST
for dt, lg in ((torch.float32, 24), (torch.float64, 23)):
    n = 1 << lg
    item = 4 if dt == torch.float32 else 8
    nbytes = 2 * n * item
    R = max(2, -(-(4 * 126 * 10**6) // nbytes))
    buf = [torch.empty(2 * n, dtype=dt, device="cuda").uniform_() for _ in range(R)]
    out = torch.empty(2, dtype=dt, device="cuda")
    reps = max(R, 20)
    for leaf in (13, 14, 15, 16):
        row = []
        for loader in (1, 8, 6):
            for split in (1, 2, 4):
                if loader == 6 and split > 1:
                    continue
                L.tf_set_loader(loader)
                L.tf_set_leaf_split(split)
                us = graph_us(lambda i: tfb.reduce(M, buf[i % R][:n], buf[i % R][n:], leaf_log2=leaf, out=out), reps)
                row.append(f"L{loader}S{split}={us:.2f}")
        print(f"{str(dt)[6:]} 2^{lg} leaf 2^{leaf}: " + " ".join(row), flush=True)
    L.tf_set_loader(0)
    L.tf_set_leaf_split(0)
    del buf
    torch.cuda.empty_cache()
