"""A/B per-call latency of the blocking numpy path (run with TFB_LIB=<variant>)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402

res = []
for lg, dt in ((8, np.float64), (12, np.float64), (16, np.float32), (18, np.float64)):
    x = np.random.default_rng(lg).standard_normal(1 << lg).astype(dt)
    for _ in range(50):
        tfb.dot_twofold_fast(x, x)
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        for _ in range(200):
            tfb.dot_twofold_fast(x, x)
        best = min(best, (time.perf_counter() - t0) / 200)
    res.append(f"2^{lg} {np.dtype(dt).name}: {1e6 * best:.1f}")
print(os.path.basename(os.environ.get("TFB_LIB", "default")), " | ".join(res))
