import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1401_0248_b200 as tfb
from paper_1401_0248_b200 import _lib
from oracle import oracle as O
L = _lib.lib()
rng = np.random.default_rng(20261020)
for case in range(300):
    dt = np.float32 if rng.random() < 0.5 else np.float64
    methods = (0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)
    m = int(rng.choice(methods)); dot = bool(rng.random() < 0.6); tp = dot and m in (2, 3) and rng.random() < 0.3
    n = int(rng.choice([rng.integers(0, 64), rng.integers(64, 5000), rng.integers(5000, 300_000), rng.integers(300_000, 2_000_000)]))
    off = int(rng.integers(0, 3)); lo = 10 if dt == np.float32 else 9
    lg = int(rng.choice([0, 0, rng.integers(lo, 18)])); scale = 2.0 ** rng.integers(-30, 30)
    xh = (rng.standard_normal(n + off) * scale * 2.0 ** rng.integers(-8, 8, n + off)).astype(dt)
    yh = rng.uniform(-1, 1, n + off).astype(dt)
    loader = int(rng.choice([0, 1, 2, 3, 6, 7, 8])); tail = int(rng.choice([0, 1, 2])); split = int(rng.choice([0, 1, 2, 4]))
    if case == 142:
        break
x, y = torch.from_numpy(xh).cuda(), torch.from_numpy(yh).cuda()
want = O.emulate(m, xh[off:], yh[off:] if dot else None, lg)
print("want", want)
for ld in (8, 1, 0):
    for tl in (0, 1, 2):
        for sp in (1, 2):
            L.tf_set_loader(ld); L.tf_set_tail(tl); L.tf_set_leaf_split(sp)
            got = tfb.reduce(tfb.Method.DIRECT, x[off:], y[off:], leaf_log2=lg).cpu().numpy()
            ok = float(got[0]).hex() == float(want[0]).hex()
            print(ld, tl, sp, "OK " if ok else "BAD", got, L.tf_last_launch().decode())
