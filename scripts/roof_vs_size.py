"""Read roof vs our f32 dottf across sizes (same bytes, rotation over >= 4x L2, CUDA-graph timed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402


def graph_us(fn, reps):
    fn(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


L = _lib.lib()
torch.cuda.set_device(0)
sink = torch.zeros(1, dtype=torch.int32, device="cuda")
print("     MB   read-roof us (GB/s)    dottf us (GB/s)   ratio")
for lg in (16, 18, 20, 22, 23, 24, 25, 26, 27, 28):
    n = 1 << lg
    nbytes = n * 4 * 2
    R = max(2, -(-(4 * 126 * 10**6) // nbytes))
    buf = [torch.empty(2 * n, dtype=torch.float32, device="cuda").uniform_() for _ in range(min(R, 8))]
    buf += [buf[i % len(buf)].clone() for i in range(len(buf), R)]
    out = torch.empty(2, dtype=torch.float32, device="cuda")
    reps = max(R, 20)
    rr = graph_us(lambda i: L.tf_read_roof(buf[i % R].data_ptr(), nbytes, 4, sink.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream), reps)
    dd = graph_us(lambda i: tfb.reduce(tfb.Method.TWOFOLD_FAST, buf[i % R][:n], buf[i % R][n:], out=out), reps)
    print(f"{nbytes / 1e6:7.1f} {rr:9.2f} ({nbytes / rr / 1e3:5.0f}) {dd:12.2f} ({nbytes / dd / 1e3:5.0f})  {dd / rr:5.2f}")
    del buf
    torch.cuda.empty_cache()
