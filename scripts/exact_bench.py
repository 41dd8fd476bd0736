"""Throughput of the GPU exact oracle (tf_exact) vs the twofold kernels on the same data."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402


def dev_ms(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


torch.cuda.set_device(0)
for name, n, dt, dot in (("f64 sum 2^28", 1 << 28, torch.float64, False), ("f64 dot 2^27", 1 << 27, torch.float64, True),
                         ("f32 dot 2^28", 1 << 28, torch.float32, True), ("f64 sum illcond 2^28", 1 << 28, torch.float64, False)):
    if "illcond" in name:
        x = tfb.philox_fill("illcond", n, seed=2, total=n)
    else:
        x = tfb.philox_fill("uniform_sym", n, seed=1, stream=0, dtype=dt)
    y = tfb.philox_fill("uniform_sym", n, seed=1, stream=1, dtype=dt) if dot else None
    nbytes = n * x.element_size() * (2 if dot else 1)
    t_ex = dev_ms(lambda: tfb.exact_dot(x, y) if dot else tfb.exact_sum(x))
    t_tp = dev_ms(lambda: tfb.exact_dot(x, y, true_products=True)) if dot else None
    t_tf = dev_ms(lambda: tfb.reduce(tfb.Method.TWOFOLD_RIGOROUS, x, y))
    print(f"{name:22s} exact {t_ex:8.3f} ms ({nbytes / t_ex / 1e6:7.0f} GB/s)"
          + (f"  exact(true products) {t_tp:8.3f} ms" if t_tp else "")
          + f"  twofold-rigorous {t_tf:8.3f} ms ({nbytes / t_tf / 1e6:7.0f} GB/s)")
