"""Leaf split (result-neutral) x loader at sizes where the auto leaf count sits just above
one wave of resident CTAs (graph-replayed, rotating copies >= 4x L2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from tail_cost import graph_us  # noqa: E402

L = _lib.lib()
torch.cuda.set_device(0)
for dt, dot, lg in ((torch.float32, True, 26), (torch.float64, False, 26), (torch.float64, True, 25),
                    (torch.float32, False, 27)):
    n = 1 << lg
    item = 4 if dt == torch.float32 else 8
    nbytes = n * item * (2 if dot else 1)
    R = max(2, -(-(4 * 126 * 10**6) // nbytes))
    buf = [torch.empty(2 * n, dtype=dt, device="cuda").uniform_(-1, 1) for _ in range(R)]
    out = torch.empty(2, dtype=dt, device="cuda")
    reps = max(R, 10)
    row = []
    ref = None
    for loader in (0, 1, 8, 2, 6):
        for split in (1, 2, 4):
            if loader in (2, 6) and split > 1:
                continue
            L.tf_set_loader(loader)
            L.tf_set_leaf_split(split)
            us = graph_us(lambda i: tfb.reduce(tfb.Method.TWOFOLD_FAST, buf[i % R][:n], buf[i % R][n:] if dot else None,
                                               out=out), reps)
            v = tfb.reduce(tfb.Method.TWOFOLD_FAST, buf[0][:n], buf[0][n:] if dot else None).cpu()
            ref = v if ref is None else ref
            assert torch.equal(v, ref)
            row.append(f"L{loader}S{split}={us:.1f}")
    L.tf_set_loader(0)
    L.tf_set_leaf_split(0)
    P = n >> tfb.leaf_log2_for(dt, n)
    print(f"{str(dt)[6:]} {'dot' if dot else 'sum'} 2^{lg} ({nbytes >> 20} MiB, P={P}): " + " ".join(row), flush=True)
    del buf
    torch.cuda.empty_cache()
