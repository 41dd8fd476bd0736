"""Launch-floor and library comparison at the small/medium BASELINE sizes.

Each number: CUDA-graph replay of R calls over input copies whose total
exceeds 4x L2 (clean HBM reads), events around one replay.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402


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
    one = torch.zeros(1, device="cuda")
    print(f"tiny elementwise kernel (launch floor): {graph_us(lambda i: one.add_(1.0), 200):.2f} us")
    for name, n, dt in (("cfg2-small", 1 << 16, torch.float32), ("cfg1", 1 << 20, torch.float64),
                        ("cfg2", 1 << 24, torch.float32)):
        nbytes = n * torch.empty(0, dtype=dt).element_size() * 2
        R = max(2, -(-(4 * 126 * 10**6) // nbytes))
        xs = [tfb.philox_fill("normal", n, seed=1, stream=0, dtype=dt) for _ in range(min(R, 4))]
        ys = [tfb.philox_fill("normal", n, seed=1, stream=1, dtype=dt) for _ in range(min(R, 4))]
        xs += [xs[i % 4].clone() for i in range(len(xs), R)]
        ys += [ys[i % 4].clone() for i in range(len(ys), R)]
        out = torch.empty(2, dtype=dt, device="cuda")
        reps = max(R, 50)
        res = {
            "torch.sum(x)": graph_us(lambda i: torch.sum(xs[i % R]), reps),
            "torch.dot(x,y) (cuBLAS)": graph_us(lambda i: torch.dot(xs[i % R], ys[i % R]), reps),
            "ours direct sum": graph_us(lambda i: tfb.reduce(tfb.Method.DIRECT, xs[i % R], out=out), reps),
            "ours dottf": graph_us(lambda i: tfb.reduce(tfb.Method.TWOFOLD_FAST, xs[i % R], ys[i % R], out=out), reps),
            "ours dott": graph_us(lambda i: tfb.reduce(tfb.Method.TWOFOLD_RIGOROUS, xs[i % R], ys[i % R], out=out),
                                  reps),
        }
        for lg in (10, 11, 12, 13):
            if (1 << lg) < n:
                res[f"ours dottf leaf 2^{lg}"] = graph_us(
                    lambda i, lg=lg: tfb.reduce(tfb.Method.TWOFOLD_FAST, xs[i % R], ys[i % R], out=out, leaf_log2=lg),
                    reps)
        print(f"== {name} ({n} x {dt}), {R} rotating copies")
        for k, v in res.items():
            print(f"   {k:32s} {v:8.2f} us")


if __name__ == "__main__":
    main()
