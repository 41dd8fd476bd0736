"""A/B two library builds on the small configs via the raw C ABI (tf_reduce) + CUDA graphs."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402


def load(path):
    L = ctypes.CDLL(path)
    vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    L.tf_reduce.argtypes = [i32, i32, vp, vp, i64, i32, vp, vp, sz, vp, i64, vp]
    L.tf_reduce.restype = i32
    return L


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


torch.cuda.set_device(0)
libs = {name: load(p) for name, p in (("new", "paper_1401_0248_b200/libtwofold_b200.so"),
                                      ("old", sys.argv[1]))}
parts = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
ctrs = torch.zeros(1024, dtype=torch.int32, device="cuda")
for name, n, dt, dot in (("cfg2-small", 1 << 16, torch.float32, True), ("cfg1", 1 << 20, torch.float64, False),
                         ("cfg2", 1 << 24, torch.float32, True)):
    nbytes = n * torch.empty(0, dtype=dt).element_size() * (2 if dot else 1)
    R = max(2, -(-(4 * 126 * 10**6) // nbytes))
    xs = [tfb.philox_fill("normal", n, seed=1, stream=0, dtype=dt) for _ in range(R)]
    ys = [tfb.philox_fill("normal", n, seed=1, stream=1, dtype=dt) for _ in range(R)] if dot else [None] * R
    out = torch.empty(2, dtype=dt, device="cuda")
    code = 0 if dt == torch.float32 else 1
    for rep in range(2):
        for lname, L in libs.items():
            def f(i, L=L):
                y = ys[i % R]
                rc = L.tf_reduce(2, code, xs[i % R].data_ptr(), None if y is None else y.data_ptr(), n, 0,
                                 out.data_ptr(), parts.data_ptr(), parts.numel(), ctrs.data_ptr(), 1024,
                                 torch.cuda.current_stream().cuda_stream)
                assert rc == 0, rc
            print(f"{name:11s} {lname}: {graph_us(f, max(R, 50)):7.2f} us")
