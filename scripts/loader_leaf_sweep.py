"""Full reduce (µs, graph-replayed over rotating copies >= 4x L2) for every loader x leaf size
at the mid-size BASELINE shapes.  Question: do the TMA rings (in-flight bytes held in shared
memory, not registers) win at mid sizes once the leaves are small enough that the
one-CTA-per-SM grid is not quantised (P >> 148)?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from tail_cost import graph_us  # noqa: E402

CASES = [
    ("cfg2 f32 dottf 2^24", torch.float32, 24, True, tfb.Method.TWOFOLD_FAST, (12, 13, 14, 15)),
    ("cfg2 f32 dott 2^24", torch.float32, 24, True, tfb.Method.TWOFOLD_RIGOROUS, (12, 13, 14, 15)),
    ("f64 dottf 2^23", torch.float64, 23, True, tfb.Method.TWOFOLD_FAST, (11, 12, 13, 14)),
    ("f32 dottf 2^22", torch.float32, 22, True, tfb.Method.TWOFOLD_FAST, (11, 12, 13)),
    ("cfg1 f64 sumtf 2^20", torch.float64, 20, False, tfb.Method.TWOFOLD_FAST, (10, 11, 12)),
]
LOADERS = {1: "LDG", 8: "LDGdeep", 2: "TMA4x16", 3: "TMA8x8", 6: "TMA4x4x4", 7: "TMA4x8x3"}


def main():
    L = _lib.lib()
    torch.cuda.set_device(0)
    only = sys.argv[1:]  # optional case-name filters
    for name, dt, lg, dot, M, leaves in CASES:
        if only and not any(o in name for o in only):
            continue
        n = 1 << lg
        item = 4 if dt == torch.float32 else 8
        nops = 2 if dot else 1
        nbytes = nops * n * item
        R = max(2, -(-(4 * 126 * 10**6) // nbytes))
        buf = [torch.empty(nops * n, dtype=dt, device="cuda").uniform_() for _ in range(R)]
        out = torch.empty(2, dtype=dt, device="cuda")
        reps = max(R, 30)
        ya = (lambda i: buf[i % R][n:]) if dot else (lambda i: None)
        L.tf_set_loader(0)
        auto = graph_us(lambda i: tfb.reduce(M, buf[i % R][:n], ya(i), out=out), reps)
        print(f"{name} ({nbytes / 1e6:.1f} MB) auto {auto:.2f} us [{L.tf_last_launch().decode()}]", flush=True)
        for leaf in leaves:
            row = []
            for code, tag in LOADERS.items():
                L.tf_set_loader(code)
                us = graph_us(lambda i: tfb.reduce(M, buf[i % R][:n], ya(i), leaf_log2=leaf, out=out), reps)
                row.append(f"{tag}={us:.2f}")
            print(f"  leaf 2^{leaf} (P={n >> leaf}): " + " ".join(row), flush=True)
        L.tf_set_loader(0)
        del buf
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
