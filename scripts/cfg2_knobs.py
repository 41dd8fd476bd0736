"""cfg2 (f32 dottf 2^24, 134 MB) under every result-neutral knob: loader x leaf split x tail,
graph-replayed over rotating copies >= 4x L2; plus the read roof on the same bytes."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402
from paper_1401_0248_b200 import _lib  # noqa: E402
from tail_cost import graph_us  # noqa: E402

L = _lib.lib()
torch.cuda.set_device(0)
n = 1 << 24
R = 4
bufs = [(torch.randn(n, device="cuda"), torch.randn(n, device="cuda")) for _ in range(R)]
sink = torch.zeros(1, dtype=torch.int32, device="cuda")
cat = [torch.cat([a, b]) for a, b in bufs]
for u in (4, 16):
    us = graph_us(lambda i: L.tf_read_roof(cat[i % R].data_ptr(), 8 * n, u, sink.data_ptr(),
                                           torch.cuda.current_stream().cuda_stream), 20)
    print(f"read roof unroll {u}: {us:.2f} us", flush=True)
ref = None
for lg in (0, 13, 14, 15, 16):
    for loader in (0, 1, 8, 2, 3, 6, 7):
        for split in (1, 2, 4):
            for tail in (0, 1, 2):
                if L.tf_set_loader(loader) or L.tf_set_leaf_split(split) or L.tf_set_tail(tail):
                    continue
                try:
                    out = tfb.reduce(tfb.Method.TWOFOLD_FAST, bufs[0][0], bufs[0][1], leaf_log2=lg).cpu()
                except Exception as exc:  # an unsupported combination
                    print(f"lg {lg} loader {loader} split {split} tail {tail}: {exc}")
                    continue
                us = graph_us(lambda i: tfb.reduce(tfb.Method.TWOFOLD_FAST, bufs[i % R][0], bufs[i % R][1],
                                                   leaf_log2=lg), 20)
                print(f"lg {lg:2d} loader {loader} split {split} tail {tail}: {us:7.2f} us  "
                      f"[{L.tf_last_launch().decode()[:70]}]", flush=True)
L.tf_set_loader(0)
L.tf_set_leaf_split(0)
L.tf_set_tail(0)
