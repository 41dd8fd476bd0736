"""Small workload touching every kernel path, for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402

L = _lib.lib()
torch.cuda.set_device(0)
assert tfb.rounding_canary()
for dt in (torch.float32, torch.float64):
    for n in (1, 1000, 70_001, (1 << 19) + 3):
        x = tfb.philox_fill("uniform_sym", n, seed=1, stream=0, dtype=dt)
        y = tfb.philox_fill("uniform_sym", n, seed=1, stream=1, dtype=dt)
        for loader, tail, split in ((1, 2, 1), (1, 1, 1), (2, 1, 1), (1, 1, 2), (1, 2, 4)):
            L.tf_set_loader(loader)
            L.tf_set_tail(tail)
            L.tf_set_leaf_split(split)
            for m in tfb.Method:
                if m is tfb.Method.WIDE and dt != torch.float32:
                    continue
                tfb.reduce(m, x, y)
                tfb.reduce(m, x[1:])  # misaligned -> scalar loads
            tfb.reduce(tfb.Method.TWOFOLD_RIGOROUS, x, y, track_product=True)
        L.tf_set_loader(0), L.tf_set_tail(0), L.tf_set_leaf_split(0)
        if n <= 1000:
            tfb.reduce(tfb.Method.TWOFOLD_FAST, x, y, flavor=tfb.Flavor.sequential())
            tfb.reduce(tfb.Method.KAHAN, x, y, flavor=tfb.Flavor.unrolled(8))
        tfb.exact_dot(x, y)
        tfb.exact_sum(x, absolute=True)
    X = tfb.rows_scaled_normal(7, 5000, seed=3, stream=0, dtype=dt)
    tfb.reduce_rows(tfb.Method.TWOFOLD_FAST, X, X)
    # session 2 paths: lane-group rows (aligned 32-byte, 16-byte, element loads), the
    # bulk-copy-fed sequential flavors, shifted loads for misaligned binary32 views
    for rows, cols, off in ((300, 16, 0), (77, 1000, 0), (50, 37, 1), (9, 4100, 2)):
        base = tfb.philox_fill("uniform_sym", rows * cols + 8, seed=4, stream=0, dtype=dt)
        Xr = base[off:off + rows * cols].view(rows, cols)
        for kind in (0, 1, 2):
            L.tf_set_rows_kernel(kind)
            tfb.reduce_rows(tfb.Method.TWOFOLD_RIGOROUS, Xr, Xr)
        L.tf_set_rows_kernel(0)
    z = tfb.philox_fill("uniform_sym", 70_003, seed=5, stream=0, dtype=dt)
    for fl in (tfb.Flavor.sequential(), tfb.Flavor.unrolled(4), tfb.Flavor.unrolled(16)):
        tfb.reduce(tfb.Method.TWOFOLD_FAST, z[1:], z[1:], flavor=fl)
        tfb.reduce(tfb.Method.KAHAN, z, flavor=fl)
    for off in (1, 2, 3):
        tfb.reduce(tfb.Method.TWOFOLD_FAST, z[off:], z[off:])
    tfb.lcg_fill("mmix", 1000, 1, dt, True, offset=5)
    tfb.two_sum(np.ones(100), np.full(100, 2.0 ** -53))
    tfb.merge_pairs(tfb.Method.TWOFOLD_FAST, torch.randn(5, 2, dtype=torch.float64, device="cuda"))
torch.cuda.synchronize()
print("sanitize workload ok")
