"""Per-call latency of the blocking numpy path for small arrays (f64 dottf)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from oracle import oracle as O  # noqa: E402  (CPU restatement of the reference seq loop, for scale)

for lg in (4, 8, 10, 12, 14, 16, 18):
    n = 1 << lg
    x = np.random.default_rng(lg).standard_normal(n)
    y = np.random.default_rng(lg + 1).standard_normal(n)
    for _ in range(20):
        tfb.dot_twofold_fast(x, y)
    reps = 300
    t0 = time.perf_counter()
    for _ in range(reps):
        tfb.dot_twofold_fast(x, y)
    ours = (time.perf_counter() - t0) / reps
    t0 = time.perf_counter()
    for _ in range(reps):
        O.seq(2, x, y)
    cpu = (time.perf_counter() - t0) / reps
    print(f"n=2^{lg}: ours {1e6 * ours:7.1f} us   CPU seq loop (C restatement, 1 thread) {1e6 * cpu:8.1f} us", flush=True)
