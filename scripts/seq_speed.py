"""Sequential flavors on the GPU (seq, unroll:4): elements/s at 2^22, vs the plain one-thread
kernel (n below the ring threshold is not measured here); CUDA events, best of 3."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402


def main():
    torch.cuda.set_device(0)
    for dt in (torch.float32, torch.float64):
        n = 1 << 22
        x = torch.rand(n, dtype=dt, device="cuda")
        y = torch.rand(n, dtype=dt, device="cuda")
        for meth in (tfb.Method.TWOFOLD_FAST, tfb.Method.TWOFOLD_RIGOROUS, tfb.Method.KAHAN):
            for fl in (tfb.Flavor.sequential(), tfb.Flavor.unrolled(4), tfb.Flavor.unrolled(16)):
                for yy in (None, y):
                    tfb.reduce(meth, x, yy, flavor=fl)
                    torch.cuda.synchronize()
                    best = 1e9
                    for _ in range(3):
                        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                        e0.record()
                        tfb.reduce(meth, x, yy, flavor=fl)
                        e1.record()
                        torch.cuda.synchronize()
                        best = min(best, e0.elapsed_time(e1))
                    print(f"{str(dt)[6:]} {meth.value:17s} {str(fl):9s} {'dot' if yy is not None else 'sum'}: "
                          f"{best:8.2f} ms  {n / best / 1e6:7.3f} Gelem/s", flush=True)


if __name__ == "__main__":
    main()
