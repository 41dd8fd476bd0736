import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1401_0248_b200 as tfb
torch.cuda.set_device(0)
M = tfb.Method.TWOFOLD_FAST
for name, dt, dot in (("f64 dot", np.float64, True), ("f32 dot", np.float32, True), ("f64 sum", np.float64, False)):
    for lg in (22, 24, 26):
        n = 1 << lg
        rng = np.random.default_rng(lg)
        x = rng.standard_normal(n).astype(dt); y = rng.standard_normal(n).astype(dt) if dot else None
        f = (lambda: tfb.dot_twofold_fast(x, y, flavor="cuda")) if dot else (lambda: tfb.sum_twofold_fast(x, flavor="cuda"))
        for _ in range(3): f()
        best = 1e9
        for _ in range(7):
            t0 = time.perf_counter()
            for _ in range(3): f()
            best = min(best, (time.perf_counter() - t0) / 3)
        print(f"{name} 2^{lg} pageable numpy: {best*1e6:9.1f} us  {n/best/1e9:6.2f} Gelem/s", flush=True)
