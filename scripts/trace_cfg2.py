"""Per-CTA timeline of a mid-size reduction (cfg2: f32 dottf 2^24) from %globaltimer stamps.

Needs the tracing variant:  bash scripts/build_variant.sh trace "-DTFB_TRACE=1"
Runs graph-replayed back-to-back calls over rotating inputs (>= 4x L2) and prints, for the LAST
call of the replay, when CTAs became resident / passed griddepcontrol.wait / finished streaming /
stored their leaf pair, and the tree kernel's wait and finish, all relative to the first stamp.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1401_0248_b200/csrc/build/variants/libtfb_trace.so"
n_log2 = int(sys.argv[2]) if len(sys.argv) > 2 else 24
dt = torch.float32 if (len(sys.argv) <= 3 or sys.argv[3] == "f32") else torch.float64
L = ctypes.CDLL(lib)
vp, i64, i32, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
L.tf_reduce.argtypes = [i32, i32, vp, vp, i64, i32, vp, vp, sz, vp, i64, vp]
L.tf_reduce.restype = i32
L.tf_trace_buffer.argtypes = [vp]
torch.cuda.set_device(0)
n = 1 << n_log2
nbytes = n * torch.empty(0, dtype=dt).element_size() * 2
R = max(2, -(-(4 * 126 * 10**6) // nbytes))
xs = [tfb.philox_fill("normal", n, seed=1, stream=0, dtype=dt) for _ in range(R)]
ys = [tfb.philox_fill("normal", n, seed=1, stream=1, dtype=dt) for _ in range(R)]
out = torch.empty(2, dtype=dt, device="cuda")
parts = torch.empty(64 << 20, dtype=torch.uint8, device="cuda")
ctrs = torch.zeros(1024, dtype=torch.int32, device="cuda")
trace = torch.zeros(8 * 4104, dtype=torch.int64, device="cuda")
code = 0 if dt == torch.float32 else 1


def f(i):
    rc = L.tf_reduce(2, code, xs[i % R].data_ptr(), ys[i % R].data_ptr(), n, 0, out.data_ptr(), parts.data_ptr(),
                     parts.numel(), ctrs.data_ptr(), 1024, torch.cuda.current_stream().cuda_stream)
    assert rc == 0, rc


reps = max(R, 40)
f(0)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(reps):
        f(i)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print(f"untraced pointer (null): {e0.elapsed_time(e1) * 1e3 / reps:.2f} us / call")
assert L.tf_trace_buffer(trace.data_ptr()) == 0
e0.record()
g.replay()
e1.record()
torch.cuda.synchronize()
print(f"traced: {e0.elapsed_time(e1) * 1e3 / reps:.2f} us / call")
t = trace.cpu().numpy().reshape(-1, 8).astype(np.int64)
ctas = int((t[:4096, 0] != 0).sum())
c = t[:ctas]
tree = t[4096]
t0 = min(c[:, 0].min(), tree[0])
q = lambda v: "min %7.2f  p10 %7.2f  med %7.2f  p90 %7.2f  max %7.2f" % tuple(
    (np.percentile(v, p) - t0) / 1e3 for p in (0, 10, 50, 90, 100))
print(f"{ctas} leaf CTAs; us relative to the first stamp of the last call")
print("resident (entry)      ", q(c[:, 0]))
print("past griddep wait     ", q(c[:, 1]))
print("streaming done        ", q(c[:, 2]))
print("leaf pair stored      ", q(c[:, 3]))
print("stream time per CTA   ", "min %7.2f  med %7.2f  max %7.2f" % tuple(
    np.percentile(c[:, 2] - c[:, 1], p) / 1e3 for p in (0, 50, 100)))
print("leaf tree per CTA     ", "min %7.2f  med %7.2f  max %7.2f" % tuple(
    np.percentile(c[:, 3] - c[:, 2], p) / 1e3 for p in (0, 50, 100)))
print("tree kernel: resident %.2f  past wait %.2f  done %.2f" % tuple((tree[:3] - t0) / 1e3))
print("last leaf stored -> tree past wait: %.2f us; tree work: %.2f us" % (
    (tree[1] - c[:, 3].max()) / 1e3, (tree[2] - tree[1]) / 1e3))
sm = c[:, 4]
per_sm = np.bincount(sm.astype(np.int64), minlength=148)
stream = (c[:, 2] - c[:, 1]) / 1e3
for k in sorted(set(per_sm[per_sm > 0])):
    sel = np.isin(sm, np.nonzero(per_sm == k)[0])
    print(f"SMs hosting {k} CTAs: {int((per_sm == k).sum()):3d} SMs, stream time per CTA med {np.median(stream[sel]):6.2f} "
          f"min {stream[sel].min():6.2f} max {stream[sel].max():6.2f} us; done at med {np.median(c[sel, 2] - t0) / 1e3:6.2f}")
