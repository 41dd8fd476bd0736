"""Where the non-streaming time of a mid-size reduction goes: read roof vs leaves-only
(tf_reduce_leaves, no tree) vs full reduce (PDL tail / ticket tail), graph-replayed
over rotating copies (>= 4x L2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
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
    best = 1e9
    for _ in range(3):
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


def main():
    L = _lib.lib()
    torch.cuda.set_device(0)
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    M = tfb.Method.TWOFOLD_FAST
    for dt, lg in ((torch.float32, 22), (torch.float32, 24), (torch.float64, 24), (torch.float32, 26)):
        n = 1 << lg
        item = 4 if dt == torch.float32 else 8
        nbytes = 2 * n * item
        R = max(2, -(-(4 * 126 * 10**6) // nbytes))
        buf = [torch.empty(2 * n, dtype=dt, device="cuda").uniform_() for _ in range(R)]
        out = torch.empty(2, dtype=dt, device="cuda")
        P = -(-n // (1 << tfb.leaf_log2_for(dt, n)))
        parts = torch.empty(P * 2 * item * 4, dtype=torch.uint8, device="cuda")
        s = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
        code = 0 if dt == torch.float32 else 1
        reps = max(R, 20)
        rr = graph_us(lambda i: L.tf_read_roof(buf[i % R].data_ptr(), nbytes, 4, sink.data_ptr(), s()), reps)
        lv = graph_us(lambda i: L.tf_reduce_leaves(2, code, buf[i % R].data_ptr(), buf[i % R][n:].data_ptr(), n, 0,
                                                   parts.data_ptr(), s()), reps)
        res = {}
        for tail in (2, 1):
            L.tf_set_tail(tail)
            res[tail] = graph_us(lambda i: tfb.reduce(M, buf[i % R][:n], buf[i % R][n:], out=out), reps)
        L.tf_set_tail(0)
        tr = graph_us(lambda i: L.tf_merge_tree(2, code, parts.data_ptr(), P, out.data_ptr(), s()), 50)
        print(f"{str(dt)[6:]} dot 2^{lg} ({nbytes / 1e6:.0f} MB, P={P}): read roof {rr:.2f} us | leaves only {lv:.2f} | "
              f"full PDL {res[2]:.2f} | full ticket {res[1]:.2f} | tree alone {tr:.2f}", flush=True)
        del buf
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
