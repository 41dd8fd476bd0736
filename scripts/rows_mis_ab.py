"""A/B of the row kernels on misaligned pitches: rows_short_kernel's lane blocks with
selects (tf_set_rows_kernel(2)) vs rows_mis_kernel's coalesced shifted vectors (3) vs a
CTA per row (1); bit-identity checked on every shape.  Kernel µs, graph-replayed over
rotating copies >= 4x L2."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from tail_cost import graph_us  # noqa: E402

SHAPES = [(100003, 777), (1 << 22, 17), (1 << 20, 63), (262144, 255), (131072, 513), (65536, 1001), (16384, 4099),
          (262144, 256)]


def main():
    L = _lib.lib()
    torch.cuda.set_device(0)
    M = tfb.Method.TWOFOLD_FAST
    for dt in (torch.float32, torch.float64):
        for rows, cols in SHAPES:
            if dt == torch.float64:
                rows //= 2
            item = torch.empty(0, dtype=dt).element_size()
            nbytes = 2 * rows * cols * item
            R = max(2, -(-(4 * 126 * 10**6) // nbytes))
            bufs = [(torch.rand(rows, cols, dtype=dt, device="cuda"), torch.rand(rows, cols, dtype=dt, device="cuda"))
                    for _ in range(R)]
            line, ref = [], None
            for kind in (2, 1, 0):
                L.tf_set_rows_kernel(kind)
                got = tfb.reduce_rows(M, bufs[0][0], bufs[0][1]).cpu()
                if ref is None:
                    ref = got
                same = torch.equal(got.view(torch.int64 if item == 8 else torch.int32),
                                   ref.view(torch.int64 if item == 8 else torch.int32))
                us = graph_us(lambda i: tfb.reduce_rows(M, bufs[i % R][0], bufs[i % R][1]), max(R, 10))
                name = L.tf_last_launch().decode().split("<")[0]
                line.append(f"k{kind}:{name[:9]} {us:8.2f}us {nbytes / us / 1e3:6.0f}GB/s{'' if same else ' DIFF'}")
            L.tf_set_rows_kernel(0)
            print(f"{str(dt)[6:]} {rows:>8} x {cols:<6} {nbytes / 1e6:7.1f}MB | " + " | ".join(line), flush=True)


if __name__ == "__main__":
    main()
