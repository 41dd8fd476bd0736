"""Pin the CPU oracle (oracle/twofold_oracle.c) against the reference itself.

Fixtures: tests/golden/reference_outputs.json, produced by running the
reference package (/root/reference/pkg/src/twofold) in this container via
tests/golden/make_golden.py.  Every oracle function that later judges the
GPU path is checked here bit-for-bit first.
"""

from fractions import Fraction

import numpy as np
import pytest

from golden_inputs import load_inputs, sha

METHOD_ID = {"direct": 0, "wide": 1, "twofold-fast": 2, "twofold-rigorous": 3, "kahan": 4}
EPS64 = 2.0 ** -53
EPS32 = 2.0 ** -24


@pytest.fixture(scope="module")
def inputs(oracle, golden):
    return load_inputs(oracle, golden)


def test_inputs_rebuilt_bit_identically(golden, inputs):
    # the oracle's LCG restatement (lcg.py:75-116) and the Philox host twin
    # rebuild exactly the bytes the reference consumed
    for name, rec in golden["inputs"].items():
        x, y = inputs[name]
        assert sha(x) == rec["x_sha256"], name
        if rec["y_sha256"] is not None:
            assert sha(y) == rec["y_sha256"], name


def test_lcg_fill_restatement(oracle, golden):
    for key, pin in golden["lcg"].items():
        kind, dt, interval = key.split("_")
        a = oracle.lcg_fill(kind, pin["n"], pin["seed"], np.float32 if dt == "f32" else np.float64,
                            interval == "sym")
        assert sha(a) == pin["sha256"], key
        assert [float(v).hex() for v in a[:4]] == pin["head"], key


def _flavor_lanes(flavor, dtype):
    kind, _, arg = flavor.partition(":")
    if kind == "seq":
        return 0
    if arg:
        return int(arg)
    return 8 if np.dtype(dtype) == np.float32 else 4  # kernels.py:54


def test_seq_and_lane_kernels_bit_exact(oracle, golden, inputs):
    """Oracle seq/unroll/vec == reference run_flavor, field for field, bitwise."""
    checked = 0
    for case in golden["cases"]:
        x, y = inputs[case["input"]]
        m = METHOD_ID[case["method"]]
        k = _flavor_lanes(case["flavor"], x.dtype)
        v, e = oracle.seq(m, x, y) if k == 0 else oracle.lanes(m, x, y, k)
        if m in (0, 1, 4):
            e = type(v)(0)  # reference reports error 0 for non-twofold methods
        assert float(v).hex() == case["value"], case
        assert float(e).hex() == case["error"], case
        checked += 1
    assert checked == len(golden["cases"]) > 1500


def test_exact_oracle_components(oracle, golden, inputs):
    """tfo_exact == expansion.exact_sum of the identical addends, component for component."""
    for name, rec in golden["inputs"].items():
        x, y = inputs[name]
        comps = oracle.exact_components(x, y)
        assert [c.hex() for c in comps] == rec["exact"], name


def test_hours100_goldens(oracle, golden):
    """accuracy.run_hours100 (accuracy.py:106-136) reproduced from the oracle's seq kernels,
    against both the fixture and the reference test's published values
    (test_acceptance.py:51-55, README.md:86-92)."""
    data = np.full(3_600_000, np.float32(0.1), np.float32)
    rows = {r["method"]: r for r in golden["hours100"]}
    d = float(oracle.seq(0, data)[0]) / 3600.0
    w = float(oracle.seq(1, data)[0]) / 3600.0
    k = float(oracle.seq(4, data)[0]) / 3600.0
    tv, te = oracle.seq(2, data)
    t = (float(tv) + float(te)) / 3600.0
    assert d.hex() == rows["direct"]["result_hours"]
    assert w.hex() == rows["wide"]["result_hours"]
    assert k.hex() == rows["kahan"]["result_hours"]
    assert t.hex() == rows["twofold-fast"]["result_hours"]
    assert (float(te) / 3600.0).hex() == rows["twofold-fast"]["estimate_hours"]
    assert abs(d - 96.3958) <= 0.0005 and abs(t - 99.9359) <= 0.001
    assert abs(float(te) / 3600.0 - 3.54008) <= 0.01


def test_reference_kats(oracle):
    """test_kernels.py:53-93 known answers, via the oracle's seq kernels."""
    x = np.array([1.0, EPS64, EPS64])
    assert oracle.seq(0, x) == (1.0, 0.0)
    assert oracle.seq(2, x) == (1.0, 2 * EPS64)
    assert oracle.seq(3, x) == (1.0, 2 * EPS64)
    assert oracle.seq(3, np.array([EPS64, 1.0])) == (1.0, EPS64)
    assert oracle.seq(4, np.array([1.0, EPS64, EPS64, -1.0]))[0] == 2 * EPS64
    r = oracle.seq(1, np.array([1.0, 2.0 ** -24], np.float32))
    assert isinstance(r[0], np.float64) and r[0] == 1.0 + 2.0 ** -24
    xl = np.array([1.0, EPS64] * 4)
    v, e = oracle.lanes(3, xl, None, 2)
    assert Fraction(float(v)) + Fraction(float(e)) == sum(Fraction(float(t)) for t in xl)


def test_philox_known_answers(oracle):
    """Random123 Philox4x32-10 known-answer vectors (kat_vectors)."""
    assert oracle.philox((0, 0, 0, 0), (0, 0)) == (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)
    assert oracle.philox((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2) == (0x408F276D, 0x41C83B0E, 0xA20BC7C6,
                                                                    0x6D5451FD)
    assert oracle.philox((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0)) == (
        0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)


def test_feistel_is_a_bijection(oracle):
    for total in (1, 2, 3, 5, 16, 100, 1000, 4096):
        img = sorted(oracle.feistel(p, total, 2) for p in range(total))
        assert img == list(range(total)), total


def test_illcond_layout_cancels_exactly(oracle):
    """cfg3 construction: +-b_k pairs cancel, so S = exact sum of the small half."""
    n = 1 << 14
    x = oracle.philox_fill("illcond", n, 2, 0, total=n)
    big = x[np.abs(x) >= 1e8]
    small = x[np.abs(x) < 1e8]
    assert len(big) == n // 2 and len(small) == n // 2
    assert sorted(big[big > 0].tolist()) == sorted((-big[big < 0]).tolist())
    assert oracle.exact(x) == oracle.exact(small)
    assert np.all((big >= 1e8) & (big < 1e9) | (big <= -1e8) & (big > -1e9))


def test_threads_baseline_matches_seq_for_one_thread(oracle, inputs):
    x, y = inputs["dot_f64_100003"]
    for m in range(5):
        if m == 1:
            continue
        assert oracle.threads(m, x, y, 1) == oracle.seq(m, x, y)


def test_threads_baseline_tracks_exact(oracle, inputs):
    x, y = inputs["dot_f64_100003"]
    S = oracle.exact(x, y)
    A = oracle.abs_sum(x, y)
    for nt in (2, 3, 8):
        v, e = oracle.threads(3, x, y, nt)
        assert oracle.deviation(v, e, S) <= oracle.bound(3, np.float64, len(x), A)


def test_non_finite_seq_and_lanes_match_reference(oracle, golden):
    """inf / -inf / NaN / overflow inputs: the oracle's seq and lane kernels propagate
    exactly as the reference's run_flavor (every NaN equal to every NaN)."""
    from golden_inputs import load_inputs
    inputs = load_inputs(oracle, golden, "nonfinite")
    for case in golden["nonfinite"]["cases"]:
        x, y = inputs[case["input"]]
        m = METHOD_ID[case["method"]]
        k = _flavor_lanes(case["flavor"], x.dtype)
        with np.errstate(all="ignore"):
            v, e = oracle.seq(m, x, y) if k == 0 else oracle.lanes(m, x, y, k)
        if m in (0, 1, 4):
            e = type(v)(0)
        assert float(v).hex() == case["value"] and float(e).hex() == case["error"], case
    assert len(golden["nonfinite"]["cases"]) == 324
