import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1401_0248_b200 as tfb
from paper_1401_0248_b200 import _lib
L = _lib.lib()
torch.cuda.set_device(0)
n = 1 << 22
x = torch.rand(n, dtype=torch.float64, device="cuda"); y = torch.rand(n, dtype=torch.float64, device="cuda")
for loader in (0, 1, 3, 7):
    L.tf_set_loader(loader)
    for m in (tfb.Method.DIRECT, tfb.Method.TWOFOLD_FAST):
        for _ in range(5): tfb.reduce(m, x, y)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(20): tfb.reduce(m, x, y)
        g.replay(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
        print(f"hot f64 dot 2^22 loader {loader} {m.value}: {e0.elapsed_time(e1)*1e3/20:.2f} us  [{L.tf_last_launch().decode()[:40]}]")
