"""Speed and bits of the oracle's C port of the seq recurrence vs the reference's
numba kernels, single thread, same arrays (this container only: it imports
/root/reference).  The CPU baselines in bench.py time the port, so it must run
at the reference's own speed.  Output: profiles/r02_cpu_port_vs_numba.txt."""
import os
import sys
import time

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_ref")
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import twofold as ref  # noqa: E402

from oracle import oracle as O  # noqa: E402

os.sched_setaffinity(0, {min(os.sched_getaffinity(0))})
n = 1 << 22
x = O.philox_fill("uniform01", n, 0, 0, 0, np.float64)
y = O.philox_fill("uniform_sym", n, 4, 1, 0, np.float64)
xf, yf = x.astype(np.float32), y.astype(np.float32)
print(f"n = {n}, one pinned core, best of 10; ns/element (reference numba | oracle C port); bits identical")
for m, mm in ((0, ref.Method.DIRECT), (1, ref.Method.WIDE), (2, ref.Method.TWOFOLD_FAST),
              (3, ref.Method.TWOFOLD_RIGOROUS), (4, ref.Method.KAHAN)):
    for a, b, tag in ((x, None, "f64 sum"), (x, y, "f64 dot"), (xf, None, "f32 sum"), (xf, yf, "f32 dot")):
        if mm is ref.Method.WIDE and a.dtype == np.float64:
            continue
        r1 = ref.run_flavor(mm, ref.Flavor.sequential(), a, b)
        r2 = O.seq(m, a, b)
        same = float(r1.value) == float(r2[0]) and (mm is ref.Method.KAHAN or float(r1.error) == float(r2[1]))
        ts = []
        for fn in (lambda: ref.run_flavor(mm, ref.Flavor.sequential(), a, b), lambda: O.seq(m, a, b)):
            fn()
            best = 1e9
            for _ in range(10):
                t0 = time.perf_counter()
                fn()
                best = min(best, time.perf_counter() - t0)
            ts.append(best * 1e9 / n)
        print(f"{mm.value:17s} {tag}: {ts[0]:6.3f} | {ts[1]:6.3f}  ratio {ts[1] / ts[0]:.2f}  bits {'same' if same else 'DIFFER'}")
