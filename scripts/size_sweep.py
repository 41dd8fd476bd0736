"""Kernel time vs size (f32 dot and f64 sum), rotation over >= 4x L2: fit t = a + bytes / BW."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
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


def main():
    torch.cuda.set_device(0)
    L = _lib.lib()
    for dt, dot, meth in ((torch.float32, True, tfb.Method.TWOFOLD_FAST), (torch.float64, False, tfb.Method.TWOFOLD_RIGOROUS)):
        pts = []
        for lg in range(16, 29):
            n = 1 << lg
            item = torch.empty(0, dtype=dt).element_size()
            nbytes = n * item * (2 if dot else 1)
            if nbytes > 8 << 30:
                break
            R = max(1, -(-(4 * 126 * 10**6) // nbytes))
            base_x = tfb.philox_fill("uniform_sym", n, seed=1, stream=0, dtype=dt)
            base_y = tfb.philox_fill("uniform_sym", n, seed=1, stream=1, dtype=dt) if dot else None
            xs = [base_x] + [base_x.clone() for _ in range(R - 1)]
            ys = [base_y] + [base_y.clone() for _ in range(R - 1)] if dot else [None] * R
            out = torch.empty(2, dtype=dt, device="cuda")
            row = [n, nbytes]
            for loader in (1, 2):
                L.tf_set_loader(loader)
                us = graph_us(lambda i: tfb.reduce(meth, xs[i % R], ys[i % R], out=out), max(R, 20))
                row.append(us)
            L.tf_set_loader(0)
            pts.append(row)
            del xs, ys
            torch.cuda.empty_cache()
        print(f"== {meth.value} {'dot' if dot else 'sum'} {dt}")
        print("      n        MB   LDG us   TMA us   LDG GB/s  TMA GB/s")
        for n, nb, a, b in pts:
            print(f"{n:10d} {nb / 1e6:9.1f} {a:8.2f} {b:8.2f} {nb / a / 1e3:9.0f} {nb / b / 1e3:9.0f}")
        big = [(nb, a) for n, nb, a, b in pts if nb >= 64e6]
        A = np.array([[1.0, nb] for nb, _ in big])
        t = np.array([a for _, a in big])
        (a0, slope), *_ = np.linalg.lstsq(A, t, rcond=None)
        print(f"LDG fit (>= 64 MB): t = {a0:.2f} us + bytes / {1e-3 / slope:.0f} GB/s")


if __name__ == "__main__":
    main()
