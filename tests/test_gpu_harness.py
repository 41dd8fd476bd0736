"""The reference's harness experiments on the GPU path (accuracy.py, bench.py
methodology; test_acceptance.py criteria C1, C4, C5, C7 adapted to the grid flavor)."""

from fractions import Fraction

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def H(cuda):
    from paper_1401_0248_b200 import harness
    return harness


def test_hours100_seq_goldens_and_grid(H):
    """C1 (test_acceptance.py:46-60): the seq flavor reproduces the goldens on the GPU."""
    import paper_1401_0248_b200 as tfb
    rows = {r.method: r for r in H.run_hours100(tfb.Flavor.sequential())}
    assert abs(rows["direct"].result_hours - 96.3958) <= 0.0005
    assert rows["kahan"].deviation_hours < 1e-5
    assert rows["wide"].deviation_hours <= 1.5e-6
    assert abs(rows["twofold-fast"].result_hours - 99.9359) <= 0.001
    assert abs(rows["twofold-fast"].estimate_hours - 3.54008) <= 0.01
    grid = {r.method: r for r in H.run_hours100(tfb.Flavor.cuda())}
    assert grid["twofold-fast"].deviation_hours <= 1.5e-6 and grid["kahan"].deviation_hours < 1e-5


def test_accuracy_bands_default_wrappers_c4(H, cuda):
    """C4 exactly as the reference states it (test_acceptance.py:133-164), through the
    package's DEFAULT wrappers (the seq flavor): f32 bands 1e-8 <= direct <= 1e-3,
    kahan <= 1e-7, twofold <= 1e-9; f64 twofold-fast v+e within 1e-30 of the exact
    sum, judged in rationals; and under 30 s."""
    import time
    import paper_1401_0248_b200 as tfb
    t0 = time.perf_counter()
    for gen in tfb.LcgKind:
        for sym in (False, True):
            x = tfb.fill(gen, 1_000_000, 1, np.float32, sym=sym)
            ref = tfb.exact_sum(x)
            rel_d = abs(tfb.relative_error(float(np.float64(tfb.sum_direct(x).value)), ref))
            kah = tfb.run_flavor(tfb.Method.KAHAN, tfb.Flavor.sequential(), x)
            rel_k = abs(tfb.relative_error(float(np.float64(kah.value)), ref))
            tf = tfb.sum_twofold_fast(x)
            rel_t = abs(tfb.relative_error(float(np.float64(tf.value)) + float(np.float64(tf.error)), ref))
            assert 1e-8 <= rel_d <= 1e-3 and rel_k <= 1e-7 and rel_t <= 1e-9, (gen, sym, rel_d, rel_k, rel_t)
        x = tfb.fill(gen, 1_000_000, 1, np.float64)
        ref_q = sum((Fraction(c) for c in tfb.exact_sum(x).components), Fraction(0))
        tf = tfb.sum_twofold_fast(x)
        assert abs((Fraction(float(tf.value)) + Fraction(float(tf.error)) - ref_q) / ref_q) <= Fraction(1, 10 ** 30)
    assert time.perf_counter() - t0 < 30.0


def test_accuracy_bands_grid_flavor(H):
    """C4 (test_acceptance.py:133-164) upper bands on the grid flavor (a tree sum is
    more accurate than sequential, so the direct lower band does not apply)."""
    import paper_1401_0248_b200 as tfb
    cuda_fl = tfb.Flavor.cuda()
    rows = H.run_accuracy_table(n=1_000_000, flavor=cuda_fl)
    for r in rows:
        if r.precision == "f32":
            limit = {"direct": 1e-3, "kahan": 1e-7, "twofold-fast": 1e-9}[r.method]
            assert abs(r.rel_error) <= limit, r
    # binary64, judged in rationals: the reference's 1e-30 criterion is met by the
    # rigorous grid flavor (and by seq, bit-identical to the reference).  The fast
    # variant loses Dekker's precondition at chain starts (|s| < |y|), like the
    # reference's own lane flavors (unroll:4 gives 1.1e-22 here): it is held to the
    # calibrated tolerance instead.
    eps = Fraction(2.0 ** -53)
    for gen in ("nr", "mmix"):
        x = tfb.lcg_fill(gen, 1_000_000, 1, torch.float64)
        ref = tfb.exact_sum(x).fraction()
        A = tfb.exact_sum(x, absolute=True).fraction()
        r = tfb.sum_twofold_rigorous(x, flavor=cuda_fl)
        assert abs((Fraction(float(r.value)) + Fraction(float(r.error)) - ref) / ref) <= Fraction(1, 10 ** 30)
        f = tfb.sum_twofold_fast(x, flavor=cuda_fl)
        D = abs(Fraction(float(f.value)) + Fraction(float(f.error)) - ref)
        assert D <= 2 * 10 ** 6 * eps * eps * A + eps * A / 64
        s = tfb.run_flavor(tfb.Method.TWOFOLD_FAST, tfb.Flavor.sequential(), x)
        assert abs((Fraction(float(s.value)) + Fraction(float(s.error)) - ref) / ref) <= Fraction(1, 10 ** 30)


def test_scaling_twofold_beats_direct(H):
    """C5 spirit (test_acceptance.py:167-177): twofold >= 10x better than direct at every n >= 1e4."""
    import paper_1401_0248_b200 as tfb
    pts, slopes = H.run_scaling_study(ns=(10 ** 4, 10 ** 5, 10 ** 6), trials=10, flavor=tfb.Flavor.cuda())
    by = {(n, m): e for n, m, e in pts}
    for n in (10 ** 4, 10 ** 5, 10 ** 6):
        assert by[(n, "twofold-fast")] <= by[(n, "direct")] / 10


def test_table1_orderings(H):
    """C7 orderings (test_acceptance.py:207-240): noread direct/fast and direct/rigorous
    ratios, and twofold at the read roof when memory-bound (the paper's thesis)."""
    mem = H.memory_rows(tiers=("large",), reps=5)
    nr = H.noread_rows(iters=1024, reps=3)
    cell = {(r.name, r.precision, r.tier): r.gelem_s for r in mem + nr}
    for p in ("f32", "f64"):
        assert 2 <= cell[("psum", p, "noread")] / cell[("psumtf", p, "noread")] <= 6
        assert 4 <= cell[("psum", p, "noread")] / cell[("psumt", p, "noread")] <= 10
        for name in ("sumtf", "sumt", "sumk"):
            assert cell[(name, p, "large")] >= 0.9 * cell[("sum", p, "large")], (name, p)
        for name in ("dottf", "dott", "dotk"):
            assert cell[(name, p, "large")] >= 0.9 * cell[("dot", p, "large")], (name, p)


def test_error_sign_fidelity_grid(H):
    """test_accuracy.py:54-66 on the grid flavor: whenever the value deviation is
    resolvable, the error channel has the sign of (exact - value)."""
    import math
    import paper_1401_0248_b200 as tfb
    checked = 0
    for seed in range(1, 8):
        for sym in (False, True):
            data = tfb.lcg_fill("mmix", 1_000_000, seed, torch.float32, sym)
            ref = tfb.exact_sum(data)
            r = tfb.sum_twofold_fast(data, flavor="cuda")
            rel_value = tfb.relative_error(float(np.float64(r.value)), ref)
            if abs(rel_value) > 10 * 2.0 ** -24:
                assert math.copysign(1, float(r.error)) == math.copysign(1, float(ref) - float(r.value))
                checked += 1
    # the tree sum is far more accurate than sequential, so few cases resolve;
    # also check the sign on cancellation-heavy cfg3-style data where it always does
    x = tfb.philox_fill("illcond", 1 << 22, seed=2, total=1 << 22)
    ref = tfb.exact_sum(x)
    r = tfb.sum_twofold_rigorous(x, flavor="cuda")
    assert math.copysign(1, float(r.error)) == math.copysign(1, float(ref.hi) - float(r.value))


def test_eft_ulp_bound_nonfinite_and_exact_permutation(cuda):
    """test_eft.py:74-103 (|y| <= ulp(x), non-finite propagation) on the device EFTs,
    and test_expansion.py:88-99 (permutation invariance) on the GPU exact oracle."""
    import math
    import paper_1401_0248_b200 as tfb
    rng = np.random.default_rng(9)
    a = rng.standard_normal(50_000) * 2.0 ** rng.integers(-300, 300, 50_000)
    b = rng.standard_normal(50_000) * 2.0 ** rng.integers(-300, 300, 50_000)
    x, y = tfb.two_sum(a, b)
    nz = x != 0
    assert np.all(np.abs(y[nz]) <= np.array([math.ulp(v) for v in x[nz]]))
    xi, _ = tfb.two_sum(np.array([math.inf, 1e308]), np.array([1.0, 1e308]))
    assert math.isinf(xi[0]) and not math.isfinite(xi[1])
    v = rng.uniform(-1e6, 1e6, 30_001)
    assert tfb.exact_sum(v).fraction() == tfb.exact_sum(rng.permutation(v)).fraction()
