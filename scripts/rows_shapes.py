"""Row-family throughput across shapes (f32 dottf, same total bytes): the BASELINE cfg4
shape and tall/skinny matrices.  Kernel µs (graph-replayed over rotating copies >= 4x L2),
GB/s and the launch description."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from tail_cost import graph_us  # noqa: E402

SHAPES = [(4096, 65536), (16384, 16384), (32768, 8192), (65536, 4096), (262144, 1024), (1 << 20, 256), (1 << 21, 128), (1 << 22, 64),
          (1 << 23, 32), (1 << 24, 16), (1 << 20, 1000), (100003, 777),
          (1 << 22, 17), (1 << 20, 63), (262144, 255), (131072, 513), (65536, 5001), (16384, 20001)]


def main():
    L = _lib.lib()
    torch.cuda.set_device(0)
    loader = int(sys.argv[1]) if len(sys.argv) > 1 else 0  # 0 = auto, 1 = LDG, 2 = TMA ...
    L.tf_set_loader(loader)
    M = tfb.Method.TWOFOLD_FAST
    only = [tuple(map(int, a.split("x"))) for a in sys.argv[2:]]  # optional: ROWSxCOLS filters
    for dt in (torch.float32, torch.float64):
        for rows, cols in SHAPES:
            if only and (rows, cols) not in only:
                continue
            if dt == torch.float64:
                rows //= 2
            item = torch.empty(0, dtype=dt).element_size()
            nbytes = 2 * rows * cols * item
            R = max(2, -(-(4 * 126 * 10**6) // nbytes))
            bufs = [(torch.rand(rows, cols, dtype=dt, device="cuda"), torch.rand(rows, cols, dtype=dt, device="cuda"))
                    for _ in range(R)]
            us = graph_us(lambda i: tfb.reduce_rows(M, bufs[i % R][0], bufs[i % R][1]), max(R, 10))
            print(f"{str(dt)[6:]} {rows:>8} x {cols:<6} {nbytes / 1e6:8.1f} MB  {us:9.2f} us  {nbytes / us / 1e3:7.0f} GB/s  "
                  f"[{L.tf_last_launch().decode()}]", flush=True)
            del bufs
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
