"""Back-to-back call period (graph replay, rotating inputs >= 4x L2) of the grid reduction vs the L2 prefetch
preamble of the LDG leaves kernel (tf_set_prefetch, KiB per operand per CTA; -1 = the automatic budget rule).
Loader forced to LDG (1) unless --auto-loader.   python scripts/prefetch_sweep.py [--auto-loader] [--kb 0,8,16,...]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--auto-loader", action="store_true")
ap.add_argument("--kb", default="0,-1,4,8,16,24,32,48,64,96")
ap.add_argument("--lo", type=int, default=20)
ap.add_argument("--hi", type=int, default=30)
ap.add_argument("--loaders", default="1")
args = ap.parse_args()
torch.cuda.set_device(0)
L = _lib.lib()
kbs = [int(k) for k in args.kb.split(",")]
loaders = [int(k) for k in args.loaders.split(",")]


def period(f, reps):
    f(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            f(i)
    best = 1e9
    for _ in range(4):
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3 / reps)
    return best


for dt in (torch.float32, torch.float64):
    for dot in (False, True):
        for blog in range(args.lo, args.hi + 1):
            nbytes = 1 << blog
            n = nbytes // torch.empty(0, dtype=dt).element_size() // (2 if dot else 1)
            R = max(2, -(-(4 * 126 * 10**6) // nbytes))
            xs = [tfb.philox_fill("normal", n, seed=1, stream=0, dtype=dt) for _ in range(R)]
            ys = [tfb.philox_fill("normal", n, seed=1, stream=1, dtype=dt) for _ in range(R)] if dot else [None] * R
            out = torch.empty(2, dtype=dt, device="cuda")

            def f(i):
                tfb.reduce(tfb.Method.TWOFOLD_FAST, xs[i % R], ys[i % R], out=out)

            row = {"dtype": str(dt).split(".")[-1], "dot": dot, "bytes_log2": blog, "us": {}}
            for ld in loaders:
                L.tf_set_loader(0 if args.auto_loader else ld)
                for kb in kbs:
                    L.tf_set_prefetch(kb)
                    us = period(f, max(R, 30 if blog < 28 else 8))
                    row["us"][f"{ld}:{kb}"] = round(us, 2)
                    if kb == kbs[0]:
                        row.setdefault("launch", {})[str(ld)] = L.tf_last_launch().decode()[:90]
            L.tf_set_prefetch(-1)
            L.tf_set_loader(0)
            print(json.dumps(row), flush=True)
            del xs, ys
