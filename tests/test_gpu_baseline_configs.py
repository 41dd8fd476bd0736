"""Every BASELINE.json config at full size on the GPU, judged against exact sums.

For each config: the grid result's deviation |v+e-S| (value only for Kahan) is
held to the SURVEY.md §8(c) tolerance, and the reference's own sequential
result on the identical data (the oracle's bit-exact port of the reference
seq kernels) is reported beside it.  Exact sums come from the CPU expansion
oracle where it finishes in seconds, else from the GPU exact oracle (itself
pinned to the CPU oracle in test_gpu_parity.py).  Writes
gpurun_out/parity_report.md.
"""

import os
from fractions import Fraction

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ROWS = []


def _report():
    out = os.path.join(REPO, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    lines = ["# Parity at BASELINE sizes (B200)", "",
             "D = |v+e-S| (Kahan/direct: |v-S|), relative to A = sum|y_i|; bound = SURVEY.md §8(c);",
             "D_ref = the reference's sequential kernels on the identical data (oracle port, bit-exact).", "",
             "| config | method | n | D/A (GPU grid) | bound/A | D_ref/A (reference seq) |", "|---|---|---|---|---|---|"]
    for r in ROWS:
        lines.append("| " + " | ".join(str(c) for c in r) + " |")
    with open(os.path.join(out, "parity_report.md"), "w") as f:
        f.write("\n".join(lines) + "\n")


@pytest.fixture(scope="module")
def tfb(cuda):
    import paper_1401_0248_b200 as m
    torch.cuda.set_device(cuda)
    with m.using_flavor("cuda"):  # the wrappers on the grid flavor for this module
        yield m
    _report()


def _dev(v, e, S, twofold):
    return abs(Fraction(float(v)) + (Fraction(float(e)) if twofold else 0) - S)


def _row(cfg, name, n, D, A, bound, Dref):
    ROWS.append((cfg, name, n, f"{float(D / A):.3e}", f"{float(bound / A):.3e}",
                 "" if Dref is None else f"{float(Dref / A):.3e}"))


def _check(oracle, tfb, cfg, x, y, methods, exact_from="cpu", ref_seq=True):
    n = x.numel()
    dt = np.float32 if x.dtype == torch.float32 else np.float64
    xh = x.cpu().numpy()
    yh = None if y is None else y.cpu().numpy()
    if exact_from == "cpu":
        S, A = oracle.exact(xh, yh), oracle.abs_sum(xh, yh)
    else:
        S = (tfb.exact_sum(x) if y is None else tfb.exact_dot(x, y)).fraction()
        A = (tfb.exact_sum(x, absolute=True) if y is None else tfb.exact_dot(x, y, absolute=True)).fraction()
    for mname in methods:
        m = oracle.METHODS.index(mname)
        meth = tfb.Method(mname)
        r = tfb.reduce(meth, x, y).cpu().numpy()
        twofold = m in (2, 3)
        D = _dev(r[0], r[1], S, twofold)
        bound = oracle.bound(m, dt, n, A, chain=(1 << tfb.leaf_log2_for(x.dtype, n)) // 256 + 40)
        if m == 2 and n >= 1 << 16:
            bound = oracle.calibrated_fast_bound(dt, n, A)
        Dref = None
        if ref_seq:
            v, e = oracle.seq(m, xh, yh)
            Dref = _dev(v, e, S, twofold)
        _row(cfg, mname, n, D, A, bound, Dref)
        assert D <= bound, (cfg, mname, float(D / A), float(bound / A))


def test_cfg1(tfb, oracle):
    x = tfb.philox_fill("uniform01", 1 << 20, seed=0, stream=0)
    _check(oracle, tfb, "cfg1 f64 sumtf U[0,1)", x, None, ("twofold-fast", "twofold-rigorous", "kahan", "direct"))
    # the GPU seq flavor reproduces the reference's own cfg1 result (golden fixture) bit for bit
    r = tfb.run_flavor(tfb.Method.TWOFOLD_FAST, tfb.Flavor.sequential(), x)
    v, e = oracle.seq(2, x.cpu().numpy())
    assert float(r.value).hex() == float(v).hex() and float(r.error).hex() == float(e).hex()


def test_cfg2_and_small(tfb, oracle):
    x = tfb.philox_fill("normal", 1 << 24, seed=1, stream=0, dtype=torch.float32)
    y = tfb.philox_fill("normal", 1 << 24, seed=1, stream=1, dtype=torch.float32)
    _check(oracle, tfb, "cfg2 f32 dot N(0,1)", x, y, ("twofold-fast", "twofold-rigorous", "kahan", "direct", "wide"))
    _check(oracle, tfb, "cfg2-small f32 dot", x[: 1 << 16].contiguous(), y[: 1 << 16].contiguous(),
           ("twofold-fast", "twofold-rigorous"))


def test_cfg3_illconditioned(tfb, oracle):
    n = 1 << 28
    x = tfb.philox_fill("illcond", n, seed=2, stream=0, total=n)
    # exact sum known by construction: the +-b_k pairs cancel, S = sum of the small half
    small = x[x.abs() < 1e8]
    S_cons = tfb.exact_sum(small).fraction()
    assert tfb.exact_sum(x).fraction() == S_cons
    _check(oracle, tfb, "cfg3 f64 illcond", x, None, ("twofold-rigorous", "kahan", "twofold-fast", "direct"),
           exact_from="gpu", ref_seq=True)


def test_cfg4_rows(tfb, oracle):
    rows, cols = 4096, 65536
    X = tfb.rows_scaled_normal(rows, cols, seed=3, stream=0)
    Y = tfb.rows_scaled_normal(rows, cols, seed=3, stream=1)
    pairs = tfb.reduce_rows(tfb.Method.TWOFOLD_FAST, X, Y).cpu().numpy()
    worst = Fraction(0)
    worst_bound = Fraction(0)
    for r in range(0, rows, 64):  # 64 rows through the CPU oracle
        xh, yh = X[r].cpu().numpy(), Y[r].cpu().numpy()
        S, A = oracle.exact(xh, yh), oracle.abs_sum(xh, yh)
        D = _dev(pairs[r, 0], pairs[r, 1], S, True)
        b = oracle.calibrated_fast_bound(np.float32, cols, A)
        assert D <= b, r
        if D / A > worst:
            worst, worst_bound = D / A, b / A
    ROWS.append(("cfg4 f32 rows dottf (64 sampled rows, worst)", "twofold-fast", cols, f"{float(worst):.3e}",
                 f"{float(worst_bound):.3e}", ""))
    # every row: GPU exact oracle
    for r in range(rows):
        S = tfb.exact_dot(X[r], Y[r]).fraction()
        A = tfb.exact_dot(X[r], Y[r], absolute=True).fraction()
        assert _dev(pairs[r, 0], pairs[r, 1], S, True) <= oracle.calibrated_fast_bound(np.float32, cols, A), r


def test_cfg5_shard(tfb, oracle):
    n = 1 << 29
    x = tfb.philox_fill("uniform_sym", n, seed=4, stream=0)
    y = tfb.philox_fill("uniform_sym", n, seed=4, stream=1)
    _check(oracle, tfb, "cfg5 shard f64 dottf U[-1,1)", x, y, ("twofold-fast", "twofold-rigorous"),
           exact_from="gpu", ref_seq=True)
