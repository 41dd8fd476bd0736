"""One seq-flavor launch (for ncu): python scripts/seq_one.py [f32|f64] [fast|rigorous|direct] [sum|dot]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_0248_b200 as tfb  # noqa: E402

dt = torch.float64 if (len(sys.argv) > 1 and sys.argv[1] == "f64") else torch.float32
meth = {"fast": tfb.Method.TWOFOLD_FAST, "rigorous": tfb.Method.TWOFOLD_RIGOROUS,
        "direct": tfb.Method.DIRECT}[sys.argv[2] if len(sys.argv) > 2 else "fast"]
dot = len(sys.argv) > 3 and sys.argv[3] == "dot"
torch.cuda.set_device(0)
n = 1 << 20
x = torch.rand(n, dtype=dt, device="cuda")
y = torch.rand(n, dtype=dt, device="cuda") if dot else None
for _ in range(2):
    r = tfb.reduce(meth, x, y, flavor=tfb.Flavor.sequential())
torch.cuda.synchronize()
print("ok", r.tolist())
