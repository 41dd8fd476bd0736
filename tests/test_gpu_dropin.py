"""The drop-in surface on the GPU against the REFERENCE's own outputs
(tests/golden/reference_dropin.json, tests/golden/reference_outputs.json):
`import paper_1401_0248_b200 as twofold` behaves like `import twofold` for the
reference's callers — fill() bytes, exact_sum / exact_dot values (binary32 dots
over exact products, binary64 over rounded products), the default wrappers'
bits (seq), and the accuracy harness numbers."""

import hashlib
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
DT = {"f32": np.float32, "f64": np.float64}


@pytest.fixture(scope="module")
def dropin():
    with open(os.path.join(HERE, "golden", "reference_dropin.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def twofold(cuda):
    import paper_1401_0248_b200 as m
    torch.cuda.set_device(cuda)
    assert m.default_flavor() == m.Flavor.sequential()
    return m


def _q(comps):
    return sum((Fraction(float.fromhex(c)) for c in comps), Fraction(0))


def test_fill_reference_signature_bytes(twofold, dropin):
    """fill(kind, n, seed, dtype, sym) with the reference's positional arguments
    returns a numpy array with the reference's exact bytes (lcg.py:108-116)."""
    for f in dropin["fill"]:
        a = twofold.fill(twofold.LcgKind(f["kind"]), f["n"], f["seed"], DT[f["dtype"]], f["sym"])
        assert isinstance(a, np.ndarray) and a.dtype == DT[f["dtype"]] and a.shape == (f["n"],)
        assert hashlib.sha256(a.tobytes()).hexdigest() == f["sha256"], f
        assert [float(v).hex() for v in a[:3]] == f["head"]
    d = twofold.fill(twofold.LcgKind.MMIX, 1000, 3, np.float64, device="cuda")
    assert d.is_cuda and np.array_equal(d.cpu().numpy(), twofold.fill(twofold.LcgKind.MMIX, 1000, 3, np.float64))
    assert twofold.fill(twofold.LcgKind.MMIX, 0).shape == (0,)


def test_exact_sum_and_dot_match_reference(twofold, dropin):
    for rec in dropin["exact"]:
        dt = DT[rec["dtype"]]
        x = twofold.fill(twofold.LcgKind.MMIX, rec["n"], rec["seed"], dt, True)
        y = twofold.fill(twofold.LcgKind.NUMERICAL_RECIPES, rec["n"], rec["seed"] + 10, dt, True)
        es, ed = twofold.exact_sum(x), twofold.exact_dot(x, y)
        assert isinstance(es, twofold.Expansion)
        assert es.fraction() == _q(rec["sum"]) and sum(map(Fraction, es.components), Fraction(0)) == _q(rec["sum"])
        # expansion.py:112-126: binary32 -> exact products, binary64 -> rounded products
        assert ed.fraction() == _q(rec["dot"]), rec
        if rec["dtype"] == "f32" and rec["n"] > 1:
            rd = twofold.exact_dot(x, y, rounded_products=True).fraction()
            want = sum((Fraction(float(v)) for v in (x * y).astype(np.float32)), Fraction(0))
            assert rd == want
        # relative_error: the same formula on the leading components (expansion.py:129-140);
        # hi/lo of two equal expansions can differ by representation, so compare to 2^-40
        got = twofold.relative_error(float(twofold.sum_direct(x).value), es)
        want = float.fromhex(rec["rel_sum_direct"])
        assert abs(got - want) <= 2.0 ** -60 + 2.0 ** -40 * abs(want), (rec, got, want)


def test_default_wrappers_return_reference_seq_bits(twofold, golden, oracle):
    """The ten wrappers with no flavor == the reference's wrappers (seq) bit for bit."""
    from golden_inputs import make
    wrappers = {("sum", "direct"): twofold.sum_direct, ("sum", "wide"): twofold.sum_wide,
                ("sum", "twofold-fast"): twofold.sum_twofold_fast,
                ("sum", "twofold-rigorous"): twofold.sum_twofold_rigorous, ("sum", "kahan"): twofold.sum_kahan,
                ("dot", "direct"): twofold.dot_direct, ("dot", "wide"): twofold.dot_wide,
                ("dot", "twofold-fast"): twofold.dot_twofold_fast,
                ("dot", "twofold-rigorous"): twofold.dot_twofold_rigorous, ("dot", "kahan"): twofold.dot_kahan}
    checked = 0
    for c in golden["cases"]:
        if c["flavor"] != "seq" or c["n"] > 20_000:
            continue
        spec = golden["inputs"][c["input"]]
        x = make(oracle, spec["x"])
        y = make(oracle, spec["y"])
        fn = wrappers[(c["op"], c["method"])]
        r = fn(x) if y is None else fn(x, y)
        assert (float(r.value).hex(), float(r.error).hex()) == (c["value"], c["error"]), c
        assert type(r.value).__name__ == c["value_type"] and r.adds_performed == c["adds"]
        checked += 1
    assert checked > 250


def test_accuracy_harness_reproduces_reference(twofold, dropin):
    """accuracy.run_accuracy_table(n=100000) and run_scaling_study on the GPU seq path
    (the reference's flavor) give the reference's numbers: identical method results,
    relative errors equal up to the leading-component representation.  The
    reference's expansion is non-overlapping but not canonical, so its hi + lo can
    miss S by a third component as large as lo/2 (~2^-54 S); ours is the
    nearest-rounding decomposition.  Hence |delta| <= 2^-60 + 2^-40 |rel|."""
    from paper_1401_0248_b200 import harness
    want = {(r["precision"], r["generator"], r["interval"], r["method"]): r for r in dropin["accuracy_table"]["rows"]}
    rows = harness.run_accuracy_table(n=100_000, seed=1)
    assert len(rows) == len(want)
    for r in rows:
        w = want[(r.precision, r.generator, r.interval, r.method)]
        wv = float.fromhex(w["rel_error"])
        assert r.valid == w["valid"] and abs(r.rel_error - wv) <= 2.0 ** -60 + 2.0 ** -40 * abs(wv), (r, wv)
    st = dropin["scaling_study"]
    pts, slopes = harness.run_scaling_study(ns=tuple(st["ns"]), trials=st["trials"], seed=st["seed"])
    wm = {(r["n"], r["method"]): float.fromhex(r["median"]) for r in st["rows"]}
    for n, m, med in pts:
        assert abs(med - wm[(n, m)]) <= 2.0 ** -60 + 2.0 ** -40 * wm[(n, m)], (n, m, med, wm[(n, m)])
    for m, s in st["slopes"].items():
        assert (slopes[m] is None) == (s is None)
        if s is not None:
            assert abs(slopes[m] - float.fromhex(s)) <= 1e-9


def test_explicit_flavor_keyword_and_switch(twofold):
    x = twofold.fill(twofold.LcgKind.MMIX, 300_001, 5, np.float64, True)
    seq = twofold.sum_twofold_fast(x)
    grid = twofold.sum_twofold_fast(x, flavor="cuda")
    with twofold.using_flavor("cuda"):
        assert twofold.sum_twofold_fast(x).twofold == grid.twofold
    assert twofold.sum_twofold_fast(x).twofold == seq.twofold
    assert twofold.run_flavor(twofold.Method.TWOFOLD_FAST, twofold.Flavor.sequential(), x).twofold == seq.twofold
