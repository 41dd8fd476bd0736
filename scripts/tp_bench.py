"""TwoProduct (opt-in Dot2-style) dots vs the reference-semantics dots: device time at the
BASELINE dot sizes (graph-replayed, rotating copies >= 4x L2 where needed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from tail_cost import graph_us  # noqa: E402

torch.cuda.set_device(0)
for dt, lg in ((torch.float32, 24), (torch.float32, 28), (torch.float64, 24), (torch.float64, 29)):
    n = 1 << lg
    item = 4 if dt == torch.float32 else 8
    nbytes = 2 * n * item
    R = max(1, -(-(4 * 126 * 10**6) // nbytes))
    buf = [tfb.philox_fill("uniform_sym", 2 * n, seed=i, dtype=dt) for i in range(R)]
    out = torch.empty(2, dtype=dt, device="cuda")
    reps = max(R, 10)
    cells = []
    for m in (tfb.Method.TWOFOLD_FAST, tfb.Method.TWOFOLD_RIGOROUS):
        for tp in (False, True):
            us = graph_us(lambda i: tfb.reduce(m, buf[i % R][:n], buf[i % R][n:], out=out, track_product=tp), reps)
            cells.append(f"{m.value}{'+TP' if tp else ''} {us:.1f} us ({nbytes / us / 1e3:.0f} GB/s)")
    print(f"{str(dt)[6:]} dot 2^{lg}: " + " | ".join(cells), flush=True)
    del buf
    torch.cuda.empty_cache()
