"""1-D reductions on 16-byte misaligned views (x[1:]) vs aligned, graph-replayed, µs and GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from tail_cost import graph_us  # noqa: E402


def main():
    L = _lib.lib()
    torch.cuda.set_device(0)
    M = tfb.Method.TWOFOLD_FAST
    for dt, lg in ((torch.float32, 24), (torch.float64, 23), (torch.float64, 27), (torch.float32, 20)):
        n = 1 << lg
        item = torch.empty(0, dtype=dt).element_size()
        nbytes = 2 * n * item
        R = max(2, -(-(4 * 126 * 10**6) // nbytes))
        bufs = [(torch.rand(n + 4, dtype=dt, device="cuda"), torch.rand(n + 4, dtype=dt, device="cuda"))
                for _ in range(R)]
        for off in ((0, 1, 2, 3) if dt == torch.float32 else (0, 1)):
            us = graph_us(lambda i: tfb.reduce(M, bufs[i % R][0][off:off + n], bufs[i % R][1][off:off + n]),
                          max(R, 10))
            print(f"{str(dt)[6:]} dot 2^{lg} offset {off}: {us:9.2f} us {nbytes / us / 1e3:7.0f} GB/s "
                  f"[{L.tf_last_launch().decode()[:70]}]", flush=True)
        del bufs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
