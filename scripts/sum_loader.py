"""LDG vs TMA loaders for large sums (f64/f32, 2 and 8 GiB)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402


def dev_ms(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


L = _lib.lib()
torch.cuda.set_device(0)
for dt in (torch.float64, torch.float32):
    for gib in (1, 2, 8):
        n = (gib << 30) // torch.empty(0, dtype=dt).element_size()
        x = tfb.philox_fill("uniform_sym", n, seed=1, dtype=dt)
        for m in (tfb.Method.TWOFOLD_RIGOROUS, tfb.Method.KAHAN, tfb.Method.TWOFOLD_FAST):
            row = []
            for loader in (1, 2, 3):
                L.tf_set_loader(loader)
                ms = dev_ms(lambda: tfb.reduce(m, x))
                row.append(f"{(gib << 30) / ms / 1e6:6.0f}")
            print(f"{str(dt)[6:]:8s} {gib} GiB {m.value:17s} LDG/TMA4x16/TMA8x8 GB/s: {' '.join(row)}")
        del x
        torch.cuda.empty_cache()
L.tf_set_loader(0)
