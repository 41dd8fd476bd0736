"""The drop-in call on pageable numpy arrays (what a reference caller passes): wall time of
dot_twofold_fast(x, y, flavor="cuda") per size, hybrid host path on (default) and off
(TFB_HYBRID_THREADS=0 in a second run).  Elements/s; the host link and DRAM bound it."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402

rng = np.random.default_rng(1)
for lg in [int(a) for a in sys.argv[1:]] or (22, 24, 26, 28):
    n = 1 << lg
    x = rng.uniform(-1, 1, n)
    y = rng.uniform(-1, 1, n)
    tfb.dot_twofold_fast(x, y, flavor="cuda")
    reps = max(3, min(20, (1 << 28) // n))
    t0 = time.perf_counter()
    for _ in range(reps):
        r = tfb.dot_twofold_fast(x, y, flavor="cuda")
    dt = (time.perf_counter() - t0) / reps
    g, h = _lib.host_split(_lib.host_engine(0))
    print(f"f64 dot 2^{lg} pageable numpy: {dt * 1e3:8.2f} ms  {n / dt / 1e9:6.2f} Gelem/s  "
          f"{16 * n / dt / 1e9:6.1f} GB/s  host share {h / max(1, g + h):.2f}", flush=True)
