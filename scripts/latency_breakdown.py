"""Fixed costs of one mid-size reduction, graph-replayed over rotating copies (>= 4x L2):
an empty launch, the read roof, leaves only (tf_reduce_leaves), the full reduce with
the PDL tail and the ticket tail, and the tree kernel alone (µs per call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from tail_cost import graph_us  # noqa: E402

CASES = [("cfg1 f64 sum", torch.float64, 20, False), ("f64 sum 2^22", torch.float64, 22, False),
         ("f32 dot 2^22", torch.float32, 22, True), ("cfg2 f32 dot", torch.float32, 24, True)]


def main():
    L = _lib.lib()
    torch.cuda.set_device(0)
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    tiny = torch.zeros(4, dtype=torch.int32, device="cuda")
    empty = graph_us(lambda i: L.tf_read_roof(tiny.data_ptr(), 16, 4, sink.data_ptr(), s()), 50)
    print(f"empty launch (1184 CTAs, one vector): {empty:.2f} us", flush=True)
    M = tfb.Method.TWOFOLD_FAST
    for name, dt, lg, dot in CASES:
        n = 1 << lg
        item = 4 if dt == torch.float32 else 8
        nops = 2 if dot else 1
        nbytes = nops * n * item
        R = max(2, -(-(4 * 126 * 10**6) // nbytes))
        buf = [torch.empty(nops * n, dtype=dt, device="cuda").uniform_() for _ in range(R)]
        out = torch.empty(2, dtype=dt, device="cuda")
        P = -(-n // (1 << tfb.leaf_log2_for(dt, n)))
        parts = torch.empty(P * 2 * item * 4, dtype=torch.uint8, device="cuda")
        code = 0 if dt == torch.float32 else 1
        reps = max(R, 30)
        yp = (lambda i: buf[i % R][n:].data_ptr()) if dot else (lambda i: None)
        ya = (lambda i: buf[i % R][n:]) if dot else (lambda i: None)
        rr = graph_us(lambda i: L.tf_read_roof(buf[i % R].data_ptr(), nbytes, 4, sink.data_ptr(), s()), reps)
        lv = graph_us(lambda i: L.tf_reduce_leaves(2, code, buf[i % R].data_ptr(), yp(i), n, 0,
                                                   parts.data_ptr(), s()), reps)
        res = {}
        for tail in (2, 1):
            L.tf_set_tail(tail)
            res[tail] = graph_us(lambda i: tfb.reduce(M, buf[i % R][:n], ya(i), out=out), reps)
        L.tf_set_tail(0)
        auto = graph_us(lambda i: tfb.reduce(M, buf[i % R][:n], ya(i), out=out), reps)
        tr = graph_us(lambda i: L.tf_merge_tree(2, code, parts.data_ptr(), P, out.data_ptr(), s()), 50)
        print(f"{name} ({nbytes / 1e6:.1f} MB, P={P}): read roof {rr:.2f} | leaves only {lv:.2f} | "
              f"PDL {res[2]:.2f} | ticket {res[1]:.2f} | auto {auto:.2f} | tree alone {tr:.2f} "
              f"[{L.tf_last_launch().decode()}]", flush=True)
        del buf
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
