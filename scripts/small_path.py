"""Small inputs: single-cluster kernel (auto tail) vs the PDL and ticket tails, vs the read roof."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from tail_cost import graph_us  # noqa: E402

L = _lib.lib()
torch.cuda.set_device(0)
sink = torch.zeros(1, dtype=torch.int32, device="cuda")
for dt, dot, lg in ((torch.float32, True, 10), (torch.float32, True, 12), (torch.float32, True, 14),
                    (torch.float32, True, 16), (torch.float64, False, 15), (torch.float64, True, 15),
                    (torch.float32, False, 16), (torch.float32, True, 17)):
    n = 1 << lg
    item = 4 if dt == torch.float32 else 8
    nbytes = n * item * (2 if dot else 1)
    R = max(2, -(-(4 * 126 * 10**6) // nbytes))
    buf = [torch.empty(2 * n, dtype=dt, device="cuda").uniform_() for _ in range(min(R, 64))]
    R = len(buf)
    out = torch.empty(2, dtype=dt, device="cuda")
    reps = max(R, 50)
    rr = graph_us(lambda i: L.tf_read_roof(buf[i % R].data_ptr(), nbytes, 4, sink.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream), reps)
    res = {}
    for tail in (0, 2, 1):
        L.tf_set_tail(tail)
        res[tail] = graph_us(lambda i: tfb.reduce(tfb.Method.TWOFOLD_FAST, buf[i % R][:n],
                                                  buf[i % R][n:] if dot else None, out=out), reps)
        if tail == 0:
            launch = L.tf_last_launch().decode()
    L.tf_set_tail(0)
    print(f"{str(dt)[6:]} {'dot' if dot else 'sum'} 2^{lg} ({nbytes >> 10} KiB): read roof {rr:.2f} us | auto {res[0]:.2f} "
          f"| PDL {res[2]:.2f} | ticket {res[1]:.2f}   [{launch}]", flush=True)
