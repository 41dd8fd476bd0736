"""e2e time of one blocking call on PINNED host inputs vs size, hybrid host path on / off (TFB_HYBRID_THREADS=0 in a child
process), to place the hybrid threshold for page-locked inputs: f64 sum and f32 dot, 2^19..2^26 elements, and the same
for pageable numpy inputs.   python scripts/hybrid_threshold.py"""
import os
import subprocess
import sys

CHILD = r'''
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1401_0248_b200 as tfb
torch.cuda.set_device(0)
M = tfb.Method.TWOFOLD_FAST
for name, dt, dot in (("f64 sum", torch.float64, False), ("f32 dot", torch.float32, True), ("f64 dot", torch.float64, True)):
    for lg in range(19, 27):
        n = 1 << lg
        x = torch.empty(n, dtype=dt, pin_memory=True).uniform_(-1, 1)
        y = torch.empty(n, dtype=dt, pin_memory=True).uniform_(-1, 1) if dot else None
        xn, yn = x.numpy().copy(), (y.numpy().copy() if dot else None)   # pageable twins
        res = []
        for a, b in ((x, y), (xn, yn)):
            for _ in range(3):
                tfb.sharded_run(M, a, b, n_global=n)
            best = 1e9
            for _ in range(7):
                t0 = time.perf_counter()
                for _ in range(5):
                    tfb.sharded_run(M, a, b, n_global=n)
                best = min(best, (time.perf_counter() - t0) / 5)
            res.append(best)
        mb = n * x.element_size() / 2**20
        print(f"{name} 2^{lg} ({mb:7.1f} MiB/operand): pinned {res[0]*1e6:9.1f} us  pageable {res[1]*1e6:9.1f} us", flush=True)
'''
for env in ({"TFB_HYBRID_THREADS": "0"}, {}, {"TFB_HYBRID_MIN_MB": "1"}):
    print("#", env or "default (hybrid from 8 MiB per operand)", flush=True)
    subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, **env), check=False)
