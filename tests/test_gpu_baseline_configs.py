"""Every BASELINE.json config at full size on the GPU: bit-exact against the
oracle's restatement of the grid tree, and judged against exact sums by
criteria that can fail.

For each config and method:
  * BIT-EXACT: the GPU pair equals oracle.emulate (the C restatement of the
    reduction tree, oracle/twofold_oracle.c) at the config's FULL size —
    cfg1, cfg2, cfg2-small, cfg3 (2^28), the cfg5 2^29 shard and cfg5 in full
    (2^32, when the device has room), sampled cfg4 rows via emulate_rows;
  * RERUNS: 10 further launches are bit-identical (every loader: LDG, TMA,
    rows, cluster);
  * TOLERANCE: |v+e-S| (value only for Kahan/direct) within SURVEY.md §8(c);
  * IMPROVEMENT (discriminating at N ~ 1/eps, where the §8(c) bound collapses
    to ~2 eps A): the twofold deviation must beat the value channel alone by a
    fixed factor, D_twofold <= D_value / F — F = 1000 for rigorous; F = 20
    for the fast variant, whose error channel loses Dekker failures on
    signed data (the reference's 100x, test_kernels.py:176-186, is stated on
    same-sign NR data; measured fast gains here: 40x cfg5, 74x cfg2-small,
    77x cfg3, 1880x cfg2, median 36x over cfg4 rows) — with a negative
    control: the same pair with its error channel zeroed (or halved) must
    FAIL the criterion.
The reference's own sequential result on the identical data (the oracle's
bit-exact port of the reference seq kernels) is reported beside it.  Exact
sums come from the CPU expansion oracle where it finishes in seconds, else
from the GPU exact oracle (itself pinned to the CPU oracle in
test_gpu_parity.py).  Writes gpurun_out/parity_report.md.
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
             "D_value = |v-S| (the pair with its error channel zeroed); gain = D_value / D (twofold only);",
             "bits = GPU pair == oracle.emulate at this n, and 10 reruns identical;",
             "D_ref = the reference's sequential kernels on the identical data (oracle port, bit-exact).", "",
             "| config | method | n | D/A (GPU grid) | bound/A | D_value/A | gain | bits | D_ref/A (reference seq) |",
             "|---|---|---|---|---|---|---|---|---|"]
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


def _hex(p):
    return (float(p[0]).hex(), float(p[1]).hex())


# Improvement factors: the twofold pair must beat its own value channel by F.
GAIN = {"twofold-fast": 20, "twofold-rigorous": 1000}


def improvement_ok(v, e, S, method: str, factor: int | None = None) -> bool:
    """D(v+e) <= D(v) / F, or both exact.  The discriminating criterion at N ~ 1/eps."""
    F = factor or GAIN[method]
    d_pair = _dev(v, e, S, True)
    d_val = _dev(v, 0.0, S, False)
    if d_val == 0:
        return d_pair == 0
    return d_pair * F <= d_val


def _check(oracle, tfb, cfg, x, y, methods, exact_from="cpu", ref_seq=True, emulate=True, reruns=10,
           gains=None):
    n = x.numel()
    dt = np.float32 if x.dtype == torch.float32 else np.float64
    xh = x.cpu().numpy()
    yh = None if y is None else y.cpu().numpy()
    if exact_from == "cpu":
        S, A = oracle.exact(xh, yh), oracle.abs_sum(xh, yh)
    else:  # the addends the kernels sum: products rounded in the data precision
        S = (tfb.exact_sum(x) if y is None else tfb.exact_dot(x, y, rounded_products=True)).fraction()
        A = (tfb.exact_sum(x, absolute=True) if y is None else
             tfb.exact_dot(x, y, rounded_products=True, absolute=True)).fraction()
    for mname in methods:
        m = oracle.METHODS.index(mname)
        meth = tfb.Method(mname)
        r = tfb.reduce(meth, x, y).cpu().numpy()
        bits = ""
        if emulate:
            want = oracle.emulate(m, xh, yh)
            assert _hex(r) == _hex(want), (cfg, mname, "GPU != emulator", _hex(r), _hex(want))
            bits = "emulator"
        for _ in range(reruns):
            assert _hex(tfb.reduce(meth, x, y).cpu().numpy()) == _hex(r), (cfg, mname, "rerun differs")
        if reruns:
            bits += f"{' + ' if bits else ''}{reruns} reruns"
        twofold = m in (2, 3)
        D = _dev(r[0], r[1], S, twofold)
        d_val = _dev(r[0], 0.0, S, False)
        bound = oracle.bound(m, dt, n, A, chain=(1 << tfb.leaf_log2_for(x.dtype, n)) // 256 + 40)
        if m == 2 and n >= 1 << 16:
            bound = oracle.calibrated_fast_bound(dt, n, A)
        Dref = None
        if ref_seq:
            v, e = oracle.seq(m, xh, yh)
            Dref = _dev(v, e, S, twofold)
        gain = "" if not twofold else ("exact" if D == 0 else f"{float(d_val / D):.3g}")
        ROWS.append((cfg, mname, n, f"{float(D / A):.3e}", f"{float(bound / A):.3e}", f"{float(d_val / A):.3e}",
                     gain, bits, "" if Dref is None else f"{float(Dref / A):.3e}"))
        assert D <= bound, (cfg, mname, float(D / A), float(bound / A))
        if twofold:
            F = (gains or {}).get(mname)
            assert improvement_ok(r[0], r[1], S, mname, F), (cfg, mname, "improvement", float(d_val / max(D, 1e-300)))
            if d_val != 0:  # negative controls: a zeroed or halved error channel must be rejected
                assert not improvement_ok(r[0], 0.0, S, mname, F), (cfg, mname, "zeroed error channel accepted")
                assert not improvement_ok(r[0], float(r[1]) / 2, S, mname, F), (cfg, mname, "halved error accepted")


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
           ("twofold-fast", "twofold-rigorous", "direct"))


def test_cfg2_negative_control_zeroed_error_channel(tfb, oracle):
    """at N = 2^24 = 1/eps the §8(c) bound alone would accept a twofold
    pair whose error channel is zeroed.  The improvement criterion must not."""
    x = tfb.philox_fill("normal", 1 << 24, seed=1, stream=0, dtype=torch.float32)
    y = tfb.philox_fill("normal", 1 << 24, seed=1, stream=1, dtype=torch.float32)
    xh, yh = x.cpu().numpy(), y.cpu().numpy()
    S, A = oracle.exact(xh, yh), oracle.abs_sum(xh, yh)
    r = tfb.reduce(tfb.Method.TWOFOLD_FAST, x, y).cpu().numpy()
    bound = oracle.calibrated_fast_bound(np.float32, 1 << 24, A)
    assert _dev(r[0], 0.0, S, True) <= bound  # the weakness: the bound accepts (v, 0) ...
    assert not improvement_ok(r[0], 0.0, S, "twofold-fast")  # ... the improvement criterion rejects it
    assert improvement_ok(r[0], r[1], S, "twofold-fast")


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
    for _ in range(10):  # the rows kernel reruns bit for bit
        assert np.array_equal(tfb.reduce_rows(tfb.Method.TWOFOLD_FAST, X, Y).cpu().numpy().view(np.uint32),
                              pairs.view(np.uint32))
    # 64 sampled rows bit-exact against the emulator (the matrix's leaf size, as the kernel)
    lg = tfb.leaf_log2_for(X.dtype, rows * cols)
    sample = list(range(0, rows, 64))
    Xs, Ys = X[sample].cpu().numpy(), Y[sample].cpu().numpy()
    ev, ee = oracle.emulate_rows(2, Xs, Ys, lg)
    for k, r in enumerate(sample):
        assert _hex(pairs[r]) == _hex((ev[k], ee[k])), (r, "rows GPU != emulator")
    worst = Fraction(0)
    worst_bound = Fraction(0)
    gains = []
    for k, r in enumerate(sample):  # 64 rows through the CPU oracle
        xh, yh = Xs[k], Ys[k]
        S, A = oracle.exact(xh, yh), oracle.abs_sum(xh, yh)
        D = _dev(pairs[r, 0], pairs[r, 1], S, True)
        b = oracle.calibrated_fast_bound(np.float32, cols, A)
        assert D <= b, r
        gains.append(float(_dev(pairs[r, 0], 0.0, S, False) / D) if D else float("inf"))
        if D / A > worst:
            worst, worst_bound = D / A, b / A
    # the reference's statistical form of the improvement criterion (test_kernels.py:176-186):
    # over the rows, the median twofold deviation beats the value channel's by >= F
    assert float(np.median(gains)) >= GAIN["twofold-fast"], np.median(gains)
    ROWS.append(("cfg4 f32 rows dottf (64 sampled rows, worst)", "twofold-fast", cols, f"{float(worst):.3e}",
                 f"{float(worst_bound):.3e}", "", f"median {np.median(gains):.3g}", "emulator + 10 reruns", ""))
    # every row: GPU exact oracle (over the kernels' addends fl32(x*y))
    for r in range(rows):
        S = tfb.exact_dot(X[r], Y[r], rounded_products=True).fraction()
        A = tfb.exact_dot(X[r], Y[r], rounded_products=True, absolute=True).fraction()
        assert _dev(pairs[r, 0], pairs[r, 1], S, True) <= oracle.calibrated_fast_bound(np.float32, cols, A), r


def test_cfg5_shard(tfb, oracle):
    n = 1 << 29
    x = tfb.philox_fill("uniform_sym", n, seed=4, stream=0)
    y = tfb.philox_fill("uniform_sym", n, seed=4, stream=1)
    _check(oracle, tfb, "cfg5 shard f64 dottf U[-1,1)", x, y, ("twofold-fast", "twofold-rigorous"),
           exact_from="gpu", ref_seq=True)


def test_cfg5_full_bit_exact(tfb, oracle):
    """cfg5 exactly as BASELINE states it: 2^32 elements on one B200 (64 GiB resident),
    the TMA loader's full launch bit-identical to the emulator and over 10 reruns."""
    free, _ = torch.cuda.mem_get_info()
    if free < 80 * 2 ** 30:
        pytest.skip("needs 80 GiB of free device memory")
    n = 1 << 32
    x = tfb.philox_fill("uniform_sym", n, seed=4, stream=0)
    y = tfb.philox_fill("uniform_sym", n, seed=4, stream=1)
    try:
        _check(oracle, tfb, "cfg5 full f64 dottf U[-1,1)", x, y, ("twofold-fast",), exact_from="gpu",
               ref_seq=False)
    finally:
        del x, y
        torch.cuda.empty_cache()
