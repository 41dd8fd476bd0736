"""The drop-in surface on CPU (no GPU): every name the reference exports
(pkg/src/twofold/__init__.py:11-42) exists with the reference's host-side
semantics — the LCG scalar API and the Expansion bookkeeping are checked
against the reference's own outputs (tests/golden/reference_dropin.json,
made by tests/golden/make_golden_dropin.py) — and the wrappers' default
flavor is the reference's seq."""

import json
import os
import subprocess
import sys
from fractions import Fraction

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))

# pkg/src/twofold/__init__.py:33-42 (__all__ of the reference)
REFERENCE_ALL = [
    "Twofold", "fast_two_sum", "two_sum", "rounding_canary",
    "Expansion", "exact_sum", "exact_dot", "expansion_add", "relative_error",
    "Method", "Flavor", "SumResult", "run_flavor",
    "sum_direct", "sum_wide", "sum_twofold_fast", "sum_twofold_rigorous",
    "sum_kahan", "dot_direct", "dot_wide", "dot_twofold_fast",
    "dot_twofold_rigorous", "dot_kahan",
    "LcgKind", "LcgState", "next_raw", "uniform01", "uniform_sym", "fill",
    "__version__",
]


@pytest.fixture(scope="module")
def dropin():
    with open(os.path.join(HERE, "golden", "reference_dropin.json")) as f:
        return json.load(f)


@pytest.fixture(scope="module")
def tfb():
    import paper_1401_0248_b200 as m
    return m


def test_every_reference_name_is_exported(tfb):
    missing = [n for n in REFERENCE_ALL if not hasattr(tfb, n)]
    assert not missing, missing
    assert set(REFERENCE_ALL) <= set(tfb.__all__)


def test_lcg_scalar_api_matches_reference(tfb, dropin):
    for rec in dropin["lcg_scalar"]:
        kind = tfb.LcgKind(rec["kind"])
        seed = rec["seed"] if kind is tfb.LcgKind.MMIX else rec["seed"] & 0xFFFFFFFF
        g = tfb.LcgState(kind, seed)
        raws = []
        for _ in range(6):
            r, g = tfb.next_raw(g)
            raws.append(r)
        assert raws == rec["raws"], rec["kind"]
        for dt, npdt in (("f32", np.float32), ("f64", np.float64)):
            for fn, key in ((tfb.uniform01, "uniform01"), (tfb.uniform_sym, "uniform_sym")):
                g = tfb.LcgState(kind, seed)
                got = []
                for _ in range(4):
                    v, g = fn(g, npdt)
                    assert type(v) is npdt
                    got.append(float(v).hex())
                assert got == rec[key][dt], (rec["kind"], rec["seed"], key, dt)
    for e in dropin["lcg_edges"]:
        v = tfb.raw_to_uniform(e["raw"], tfb.LcgKind(e["kind"]), np.float32 if e["dtype"] == "f32" else np.float64,
                               e["sym"])
        assert float(v).hex() == e["value"], e


def test_lcg_state_is_immutable_and_defaults(tfb):
    g = tfb.LcgState(tfb.LcgKind.NUMERICAL_RECIPES)
    assert g.state == 1  # DEFAULT_SEED (lcg.py:31)
    _, g2 = tfb.next_raw(g)
    assert g.state == 1 and g2 is not g
    with pytest.raises(Exception):
        g.state = 5  # frozen dataclass
    assert tfb.next_raw(tfb.LcgState(tfb.LcgKind.NUMERICAL_RECIPES, 0))[0] == 1013904223
    assert tfb.next_raw(tfb.LcgState(tfb.LcgKind.MMIX, 0))[0] == 1442695040888963407


def test_expansion_add_matches_reference(tfb, dropin):
    for c in dropin["expansion_add"]:
        e = tfb.Expansion(())
        for v in c["values"]:
            e = tfb.expansion_add(e, float.fromhex(v))
        assert [x.hex() for x in e.components] == c["components"], c["values"]
        assert float(e).hex() == c["float"] and e.hi.hex() == c["hi"] and e.lo.hex() == c["lo"]
        assert e.is_zero == c["is_zero"]


def test_exact_value_is_an_expansion(tfb, dropin):
    """ExactValue (the GPU oracle's result) decomposes its limbs into a non-overlapping
    expansion equal as a rational to the reference's components, with hi = fl(S)."""
    from paper_1401_0248_b200.exact import _components_of
    for rec in dropin["exact"]:
        for key in ("sum", "dot"):
            q = sum((Fraction(float.fromhex(c)) for c in rec[key]), Fraction(0))
            comps = _components_of(q)
            assert sum((Fraction(c) for c in comps), Fraction(0)) == q
            assert comps[-1] == float(q)  # hi = fl(S)
            mags = [abs(c) for c in comps]
            assert mags == sorted(mags)
    assert issubclass(tfb.ExactValue, tfb.Expansion)
    with pytest.raises(ValueError):
        tfb.relative_error(1.0, tfb.Expansion(()))


def test_default_flavor_is_seq_and_switchable(tfb):
    assert tfb.default_flavor() == tfb.Flavor.sequential()
    with tfb.using_flavor("cuda") as fl:
        assert fl == tfb.Flavor.cuda() and tfb.default_flavor() == fl
    assert tfb.default_flavor() == tfb.Flavor.sequential()
    prev = tfb.set_default_flavor(tfb.Flavor.unrolled(4))
    try:
        assert str(tfb.default_flavor()) == "unroll:4"
    finally:
        tfb.set_default_flavor(prev)
    with pytest.raises(ValueError):
        tfb.set_default_flavor("simd")
    with pytest.raises(TypeError):
        tfb.set_default_flavor(3)


def test_default_flavor_from_environment():
    code = "import paper_1401_0248_b200 as t; print(t.default_flavor())"
    env = dict(os.environ, TWOFOLD_B200_FLAVOR="cuda", CUDA_VISIBLE_DEVICES="")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd=os.path.dirname(HERE), check=True).stdout.strip()
    assert out == "cuda"


def test_fill_validates_before_touching_a_device(tfb):
    with pytest.raises(ValueError):
        tfb.fill("pcg", 10)
    with pytest.raises(TypeError):
        tfb.fill(tfb.LcgKind.MMIX, 10, 1, np.int32)
