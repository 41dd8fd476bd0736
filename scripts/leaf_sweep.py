"""Leaf size x loader at mid sizes: for each (precision, sum/dot, n) the best time over the
loaders at leaf auto-1 / auto / auto+1 (twofold-fast), graph-replayed over rotating copies
>= 4x L2.  Output: one JSON line per case (for choosing the auto leaf rule)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from tune_loaders import graph_us  # noqa: E402

L = _lib.lib()
torch.cuda.set_device(0)
M = tfb.Method.TWOFOLD_FAST
for dt in (torch.float32, torch.float64):
    item = 4 if dt == torch.float32 else 8
    lo = 10 if dt == torch.float32 else 9
    for dot in (False, True):
        for lgn in range(19, 28):
            n = 1 << lgn
            nbytes = n * item * (2 if dot else 1)
            R = max(2, -(-(4 * 126 * 10**6) // nbytes))
            bufs = [(torch.empty(n, dtype=dt, device="cuda").uniform_(-1, 1),
                     torch.empty(n, dtype=dt, device="cuda").uniform_(-1, 1) if dot else None) for _ in range(R)]
            auto = tfb.leaf_log2_for(dt, n)
            res = {}
            for leaf in sorted({max(lo, auto - 1), auto, min(16, auto + 1)}):
                best = None
                for loader in (1, 8, 2, 3, 6, 7):
                    L.tf_set_loader(loader)
                    us = graph_us(lambda i: tfb.reduce(M, bufs[i % R][0], bufs[i % R][1], leaf_log2=leaf), max(R, 10))
                    if best is None or us < best[0]:
                        best = (us, loader)
                res[leaf] = best
            L.tf_set_loader(0)
            print(json.dumps({"dtype": str(dt)[6:], "dot": dot, "n_log2": lgn, "bytes": nbytes, "auto": auto,
                              "best_by_leaf": {str(k): v for k, v in res.items()}}), flush=True)
            del bufs
            torch.cuda.empty_cache()
