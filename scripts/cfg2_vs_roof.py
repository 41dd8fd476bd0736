"""One cfg2-sized (134 MB) launch each of tf_read_roof and dottf f32 — for an ncu side-by-side."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402

torch.cuda.set_device(0)
L = _lib.lib()
n = 1 << 24
buf = torch.empty(2 * n, dtype=torch.float32, device="cuda").uniform_()
sink = torch.zeros(1, dtype=torch.int32, device="cuda")
out = torch.empty(2, dtype=torch.float32, device="cuda")
for _ in range(2):
    L.tf_read_roof(buf.data_ptr(), 8 * n, 4, sink.data_ptr(), torch.cuda.current_stream().cuda_stream)
    tfb.reduce(tfb.Method.TWOFOLD_FAST, buf[:n], buf[n:], out=out)
torch.cuda.synchronize()
print("ok", out.tolist())
