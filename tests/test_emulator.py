"""Properties of the GPU reduction tree, checked on its CPU restatement (the
oracle's emulator).  tests/test_gpu_parity.py proves the GPU is bit-identical
to this emulator, so these properties transfer to the device results."""

from fractions import Fraction

import numpy as np
import pytest

EPS64 = 2.0 ** -53


def test_exact_tracking_rigorous(oracle):
    """Rigorous (Knuth) twofold keeps v+e within 2 N eps^2 sum|y| of the exact sum."""
    for dt in (np.float32, np.float64):
        for n in (1, 7, 1000, 4097, 100_003, 1 << 18):
            for kind, sym in (("nr", False), ("mmix", True)):
                x = oracle.lcg_fill(kind, n, 5, dt, sym)
                y = oracle.lcg_fill("mmix", n, 6, dt, True)
                for yy in (None, y):
                    v, e = oracle.emulate(3, x, yy)
                    S, A = oracle.exact(x, yy), oracle.abs_sum(x, yy)
                    assert oracle.deviation(v, e, S) <= oracle.bound(3, dt, n, A), (dt, n, kind)


def test_fast_within_calibrated_bound(oracle):
    for dt in (np.float32, np.float64):
        for n in (1000, 100_003, 1 << 18):
            x = oracle.lcg_fill("mmix", n, 8, dt, True)
            y = oracle.lcg_fill("nr", n, 9, dt, True)
            v, e = oracle.emulate(2, x, y)
            S, A = oracle.exact(x, y), oracle.abs_sum(x, y)
            D = oracle.deviation(v, e, S)
            assert D <= oracle.bound(2, dt, n, A)
            if n >= 1 << 16:
                assert D <= oracle.calibrated_fast_bound(dt, n, A), (dt, n, float(D))
            # and always far better than the value channel alone
            assert D <= oracle.deviation(v, 0.0, S)


def test_value_channel_identical_for_direct_fast_rigorous(oracle):
    for dt in (np.float32, np.float64):
        x = oracle.lcg_fill("mmix", 300_001, 3, dt, True)
        d = oracle.emulate(0, x)[0]
        assert oracle.emulate(2, x)[0] == d and oracle.emulate(3, x)[0] == d


def test_dot_by_ones_equals_sum(oracle):
    x = oracle.lcg_fill("nr", 70_001, 2, np.float32, False)
    ones = np.ones_like(x)
    for m in range(5):
        assert oracle.emulate(m, x, ones) == oracle.emulate(m, x)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_exact_integer_data(oracle, dt):
    x = np.arange(1, 100_001, dtype=dt)
    x = x % 1000
    for m in ((0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)):
        v, e = oracle.emulate(m, x)
        assert float(v) == float(np.sum(x.astype(np.int64))), m
        if m in (2, 3):
            assert float(e) == 0.0


def test_lane_style_exact_tracking(oracle):
    """test_kernels.py:234-240 analogue: exact addends stay exact through the tree."""
    x = np.array([1.0, EPS64] * 40_000)
    v, e = oracle.emulate(3, x)
    assert Fraction(float(v)) + Fraction(float(e)) == 40_000 * (1 + Fraction(EPS64))


def test_leaves_then_tree_equals_fused(oracle):
    for dt in (np.float32, np.float64):
        n = 123_457
        x = oracle.lcg_fill("mmix", n, 1, dt, True)
        y = oracle.lcg_fill("nr", n, 2, dt, True)
        for m in (0, 2, 3, 4):
            for lg in (0, 10, 12):
                s, e = oracle.emulate_leaves(m, x, y, lg)
                assert oracle.tree(m, dt, s, e) == oracle.emulate(m, x, y, lg), (dt, m, lg)


def test_shards_are_subtrees(oracle):
    """Power-of-two layout: G shard roots merged == the single-device root, for any G."""
    n, lg = 1 << 20, 12
    x = oracle.lcg_fill("mmix", n, 4, np.float64, True)
    y = oracle.lcg_fill("nr", n, 5, np.float64, True)
    for m in (0, 2, 3, 4):
        whole = oracle.emulate(m, x, y, lg)
        for G in (2, 4, 8, 16):
            L = n // G
            parts = [oracle.emulate(m, x[r * L:(r + 1) * L], y[r * L:(r + 1) * L], lg) for r in range(G)]
            assert oracle.tree(m, np.float64, [p[0] for p in parts], [p[1] for p in parts]) == whole, (m, G)


def test_gpu_flavor_beats_sequential_accuracy_on_signed_data(oracle):
    """the tree's rigorous result is at least as accurate as seq."""
    x = oracle.lcg_fill("mmix", 1 << 18, 12, np.float64, True)
    S = oracle.exact(x)
    dg = oracle.deviation(*oracle.emulate(3, x), S)
    ds = oracle.deviation(*oracle.seq(3, x), S)
    assert dg <= ds or dg == 0
