"""Tail variants on the LDG path: auto (PDL) vs ticket vs cluster-group tail (tail 3),
graph-replayed over rotating copies (>= 4x L2); every variant checked bit-identical.

Record of a rejected experiment (profiles/r01_summary.md): the cluster-group tail
(tail 3) was removed from the library after this measurement; tf_set_tail(3) now
fails and the T3 columns repeat the automatic tail."""
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
cases = [(torch.float32, True, lg) for lg in (17, 18, 20, 22, 24)] + [(torch.float64, False, 20), (torch.float64, False, 23),
                                                                      (torch.float64, True, 22)]
for dt, dot, lg in cases:
    n = 1 << lg
    item = 4 if dt == torch.float32 else 8
    nbytes = n * item * (2 if dot else 1)
    R = max(2, -(-(4 * 126 * 10**6) // nbytes))
    buf = [torch.empty(2 * n, dtype=dt, device="cuda").uniform_(-1, 1) for _ in range(min(R, 64))]
    R = len(buf)
    out = torch.empty(2, dtype=dt, device="cuda")
    reps = max(R, 30)
    res, vals = {}, {}
    for loader in (0, 1):
        L.tf_set_loader(loader)
        for tail in (0, 1, 2, 3):
            L.tf_set_tail(tail)
            fn = (lambda i: tfb.reduce(tfb.Method.TWOFOLD_FAST, buf[i % R][:n], buf[i % R][n:] if dot else None, out=out))
            res[(loader, tail)] = graph_us(fn, reps)
            vals[(loader, tail)] = tfb.reduce(tfb.Method.TWOFOLD_FAST, buf[0][:n], buf[0][n:] if dot else None).cpu()
            if tail == 3:
                launch = L.tf_last_launch().decode()
    L.tf_set_tail(0)
    L.tf_set_loader(0)
    same = all(torch.equal(v, vals[(0, 0)]) for v in vals.values())
    print(f"{str(dt)[6:]} {'dot' if dot else 'sum'} 2^{lg} ({nbytes >> 10} KiB): "
          + " ".join(f"L{l}T{t}={u:.2f}" for (l, t), u in res.items()) + f"  identical={same}  [{launch[:70]}]",
          flush=True)
    del buf
    torch.cuda.empty_cache()
