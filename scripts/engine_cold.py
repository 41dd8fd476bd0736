"""Cold cost of the first numpy call (engine creation) vs steady state."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402

torch.cuda.set_device(0)
torch.zeros(1, device="cuda")
tfb.rounding_canary()
x = np.random.default_rng(1).standard_normal(1 << 16).astype(np.float32)
t0 = time.perf_counter()
tfb.dot_twofold_fast(x, x)
t1 = time.perf_counter()
tfb.dot_twofold_fast(x, x)
t2 = time.perf_counter()
big = np.random.default_rng(2).standard_normal(1 << 24)
tfb.dot_twofold_fast(big, big)
t3 = time.perf_counter()
tfb.dot_twofold_fast(big, big)
t4 = time.perf_counter()
print(f"first small call {1e3 * (t1 - t0):.2f} ms, second {1e3 * (t2 - t1):.3f} ms; "
      f"first 2^24 f64 call {1e3 * (t3 - t2):.2f} ms, second {1e3 * (t4 - t3):.2f} ms")
