"""Where the time of one blocking host-input call goes (tf_host_reduce on small inputs)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
L = _lib.lib()
_lib.ensure_canary(0)
eng = _lib.host_engine(0)
print("engine threads", L.tf_host_engine_threads(eng))


def per_call(fn, reps=300):
    for _ in range(10):
        fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return 1e6 * (time.perf_counter() - t0) / reps


for dt, lg in ((np.float32, 16), (np.float64, 16), (np.float64, 18), (np.float64, 20)):
    n = 1 << lg
    xh = np.random.default_rng(1).standard_normal(n).astype(dt)
    yh = np.random.default_rng(2).standard_normal(n).astype(dt)
    xp, yp = torch.from_numpy(xh).pin_memory(), torch.from_numpy(yh).pin_memory()
    code = 0 if dt == np.float32 else 1
    pair = np.empty(2, dt)
    tag = f"{np.dtype(dt).name} 2^{lg} ({2 * xh.nbytes >> 10} KiB)"
    print(tag, "raw tf_host_reduce pageable: %.1f us" % per_call(
        lambda: L.tf_host_reduce(eng, 2, code, xh.ctypes.data, yh.ctypes.data, n, 0, pair.ctypes.data, None)))
    print(tag, "raw tf_host_reduce pinned:   %.1f us" % per_call(
        lambda: L.tf_host_reduce(eng, 2, code, xp.data_ptr(), yp.data_ptr(), n, 0, pair.ctypes.data, None)))
    print(tag, "public dot_twofold_fast numpy: %.1f us" % per_call(lambda: tfb.dot_twofold_fast(xh, yh)))
    xd = torch.empty(n, dtype=xp.dtype, device="cuda")
    yd = torch.empty_like(xd)

    def h2d_only():
        xd.copy_(xp, non_blocking=True)
        yd.copy_(yp, non_blocking=True)
        torch.cuda.synchronize()
    print(tag, "torch pinned H2D x2 + sync: %.1f us" % per_call(h2d_only))

    def torch_dot():
        a = torch.from_numpy(xh).cuda()
        b = torch.from_numpy(yh).cuda()
        return torch.dot(a, b).item()
    print(tag, "torch pageable .cuda() x2 + dot + item: %.1f us" % per_call(torch_dot))
    buf = np.empty_like(xh)
    print(tag, "np.copyto one operand: %.1f us" % per_call(lambda: np.copyto(buf, xh)))
    print(tag, "empty sync: %.1f us" % per_call(torch.cuda.synchronize))

for lg in (20, 24, 26):
    n = 1 << lg
    xh = np.random.default_rng(1).standard_normal(n)
    yh = np.random.default_rng(2).standard_normal(n)
    pair = np.empty(2)
    for th in (1, 2, 4, 8, 12):
        e = _lib.host_engine(0, chunk_bytes=0, threads=th)
        us = per_call(lambda: L.tf_host_reduce(e, 2, 1, xh.ctypes.data, yh.ctypes.data, n, 0, pair.ctypes.data, None),
                      reps=max(3, (1 << 27) // n))
        print(f"f64 dot 2^{lg} pageable threads={th}: {us:9.1f} us {16 * n / us / 1e3:6.2f} GB/s", flush=True)
