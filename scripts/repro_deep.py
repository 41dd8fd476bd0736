"""Deep LDG loader (UF=2) with R < U: per-leaf partials vs the emulator."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1401_0248_b200 as tfb
from paper_1401_0248_b200 import _lib
from oracle import oracle as O
L = _lib.lib()
L.tf_set_loader(8)
rng = np.random.default_rng(5)
for dt, lgs in ((np.float64, (9, 10, 11, 12)), (np.float32, (10, 11, 12, 13))):
    for lg in lgs:
        n = (1 << lg) * 37 + 5
        xh = rng.standard_normal(n).astype(dt); yh = rng.standard_normal(n).astype(dt)
        x, y = torch.from_numpy(xh).cuda(), torch.from_numpy(yh).cuda()
        P = -(-n // (1 << lg))
        parts = torch.zeros(P * 2, dtype=torch.float64 if dt == np.float64 else torch.float32, device="cuda")
        rc = L.tf_reduce_leaves(0, 1 if dt == np.float64 else 0, x.data_ptr(), y.data_ptr(), n, lg, parts.data_ptr(),
                                torch.cuda.current_stream().cuda_stream)
        print("rc", rc, L.tf_last_cuda_error().decode(), flush=True)
        torch.cuda.synchronize()
        got = parts.view(P, 2).cpu().numpy()
        ev, ee = O.emulate_leaves(0, xh, yh, lg)
        bad = [i for i in range(P) if float(got[i, 0]).hex() != float(ev[i]).hex()]
        print(np.dtype(dt).name, "lg", lg, "R", (1 << lg) // (256 * (16 // np.dtype(dt).itemsize)), "bad leaves", len(bad), bad[:5],
              "| launch:", L.tf_last_launch().decode()[:60])
        if bad:
            i = bad[0]
            print("   leaf", i, "got", got[i, 0], "want", ev[i])
