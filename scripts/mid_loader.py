"""Mid-size loaders: LDG vs TMA small-ring variants (6: 4x4KiB, 4 CTAs/SM; 7: 4x8KiB, 3 CTAs/SM)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from roof_vs_size import graph_us  # noqa: E402

L = _lib.lib()
torch.cuda.set_device(0)
sink = torch.zeros(1, dtype=torch.int32, device="cuda")
for dt, dot, meth in ((torch.float32, True, tfb.Method.TWOFOLD_FAST), (torch.float64, False, tfb.Method.TWOFOLD_FAST),
                      (torch.float64, True, tfb.Method.TWOFOLD_RIGOROUS), (torch.float32, False, tfb.Method.KAHAN)):
    print(f"== {meth.value} {'dot' if dot else 'sum'} {dt}")
    for lg in (18, 20, 22, 24, 25, 26, 27):
        n = 1 << lg
        item = torch.empty(0, dtype=dt).element_size()
        nbytes = n * item * (2 if dot else 1)
        R = max(2, -(-(4 * 126 * 10**6) // nbytes))
        buf = [torch.empty(2 * n, dtype=dt, device="cuda").uniform_() for _ in range(min(R, 8))]
        buf += [buf[i % len(buf)].clone() for i in range(len(buf), R)]
        out = torch.empty(2, dtype=dt, device="cuda")
        reps = max(R, 20)
        row = []
        rr = graph_us(lambda i: L.tf_read_roof(buf[i % R].data_ptr(), nbytes, 4, sink.data_ptr(),
                                               torch.cuda.current_stream().cuda_stream), reps)
        for loader in (1, 6, 7, 2):
            L.tf_set_loader(loader)
            us = graph_us(lambda i: tfb.reduce(meth, buf[i % R][:n], buf[i % R][n:] if dot else None, out=out), reps)
            row.append(us)
        L.tf_set_loader(0)
        print(f"{nbytes / 1e6:8.1f} MB  roof {rr:7.2f}  LDG {row[0]:7.2f}  TMA4x4K/4 {row[1]:7.2f}  TMA4x8K/3 {row[2]:7.2f}  TMA4x16K/1 {row[3]:7.2f} us")
        del buf
        torch.cuda.empty_cache()
