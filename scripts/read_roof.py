"""Practical HBM read ceiling on this B200 vs the reductions (paper read1/read2 method)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402


def dev_ms(fn, reps=20):
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
nbytes = 8 << 30
buf = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
buf.uniform_()
sink = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for u in (2, 4, 8, 16):
    ms = dev_ms(lambda: L.tf_read_roof(buf.data_ptr(), nbytes, u, sink.data_ptr(), s))
    print(f"read roof unroll {u:2d}: {ms:8.3f} ms  {nbytes / ms / 1e6:7.0f} GB/s")
cp = torch.empty_like(buf[: buf.numel() // 2])
ms = dev_ms(lambda: cp.copy_(buf[: buf.numel() // 2]))
print(f"torch copy 4 GiB -> 4 GiB: {ms:8.3f} ms  {nbytes / ms / 1e6:7.0f} GB/s (read+write)")
x, y = buf[: buf.numel() // 2], buf[buf.numel() // 2:]
for loader in (1, 2, 3, 4, 5):
    L.tf_set_loader(loader)
    ms = dev_ms(lambda: tfb.reduce(tfb.Method.TWOFOLD_FAST, x, y))
    print(f"dottf f64 8 GiB loader {loader}: {ms:8.3f} ms  {nbytes / ms / 1e6:7.0f} GB/s  {L.tf_last_launch().decode()[:60]}")
L.tf_set_loader(0)
for m in (tfb.Method.DIRECT, tfb.Method.TWOFOLD_RIGOROUS):
    ms = dev_ms(lambda: tfb.reduce(m, buf))
    print(f"{m.value} sum f64 8 GiB: {ms:8.3f} ms  {nbytes / ms / 1e6:7.0f} GB/s")
