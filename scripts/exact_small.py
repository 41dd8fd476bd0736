"""Fixed cost of the GPU exact oracle: tf_exact kernel time (CUDA events) vs n, f64 sum."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
L = _lib.lib()
recs, nbytes = ctypes.c_int64(0), ctypes.c_size_t(0)
L.tf_exact_workspace(ctypes.byref(recs), ctypes.byref(nbytes))
buf = torch.zeros(nbytes.value, dtype=torch.uint8, device="cuda")
counter = torch.zeros(1, dtype=torch.int32, device="cuda")
out = torch.empty(2, dtype=torch.float64, device="cuda")
limbs = torch.empty(80, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for lg in (10, 14, 16, 18, 20, 22, 24, 26, 28):
    n = 1 << lg
    x = tfb.philox_fill("uniform_sym", n, seed=1, stream=0, dtype=torch.float64)
    fn = lambda: L.tf_exact(1, x.data_ptr(), None, n, 0, out.data_ptr(), limbs.data_ptr(), buf.data_ptr(),  # noqa: E731
                            nbytes.value, counter.data_ptr(), s)
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e3
    print(f"f64 sum 2^{lg}: {t:9.2f} us  {8 * n / t / 1e3:7.0f} GB/s  (records {recs.value})", flush=True)
