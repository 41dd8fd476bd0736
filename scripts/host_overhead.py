"""Host-side cost of the Python API per call (no sync) and user-visible latency (with sync)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402

torch.cuda.set_device(0)
x = tfb.philox_fill("normal", 1 << 16, seed=1, dtype=torch.float32)
y = tfb.philox_fill("normal", 1 << 16, seed=2, dtype=torch.float32)
out = torch.empty(2, device="cuda")
for _ in range(100):
    tfb.reduce(tfb.Method.TWOFOLD_FAST, x, y, out=out)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N):
    tfb.reduce(tfb.Method.TWOFOLD_FAST, x, y, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"tfb.reduce (async, device tensors): {1e6 * (t1 - t0) / N:.1f} us host time per call")
tfb.dot_twofold_fast(x, y)  # warm-up (creates the host engine)
t0 = time.perf_counter()
for _ in range(200):
    r = tfb.dot_twofold_fast(x, y)
t1 = time.perf_counter()
print(f"dot_twofold_fast (device tensors, returns numpy scalars): {1e6 * (t1 - t0) / 200:.1f} us per call")
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    r = tfb.reduce(tfb.Method.TWOFOLD_FAST, x, y).cpu()
t1 = time.perf_counter()
print(f"reduce(...).cpu() (device tensors, async path + D2H): {1e6 * (t1 - t0) / 200:.1f} us per call")
xh, yh = x.cpu().numpy(), y.cpu().numpy()
t0 = time.perf_counter()
for _ in range(200):
    r = tfb.dot_twofold_fast(xh, yh)
t1 = time.perf_counter()
print(f"dot_twofold_fast (numpy 2^16 f32, H2D each call): {1e6 * (t1 - t0) / 200:.1f} us per call")
import ctypes  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
L = _lib.lib()
parts = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
ctrs = torch.zeros(64, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
args = (2, 0, x.data_ptr(), y.data_ptr(), x.numel(), 0, out.data_ptr(), parts.data_ptr(), parts.numel(), ctrs.data_ptr(), 64, s)
t0 = time.perf_counter()
for _ in range(N):
    L.tf_reduce(*args)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"raw ctypes tf_reduce: {1e6 * (t1 - t0) / N:.1f} us host time per call")

# Host-buffer engine throughput over sizes (numpy pageable and pinned inputs, f64 dot).
for lg in (16, 20, 24, 27):
    n = 1 << lg
    xh = np.random.default_rng(lg).standard_normal(n)
    yh = np.random.default_rng(lg + 1).standard_normal(n)
    reps = max(3, min(200, (1 << 26) // n))
    for kind in ("pageable", "pinned"):
        xa, ya = (xh, yh) if kind == "pageable" else (torch.from_numpy(xh).pin_memory(), torch.from_numpy(yh).pin_memory())
        tfb.dot_twofold_fast(xa, ya)
        t0 = time.perf_counter()
        for _ in range(reps):
            r = tfb.dot_twofold_fast(xa, ya)
        dt = (time.perf_counter() - t0) / reps
        print(f"dot_twofold_fast f64 2^{lg} {kind:8s}: {1e6 * dt:9.1f} us  {16 * n / dt / 1e9:6.2f} GB/s", flush=True)
