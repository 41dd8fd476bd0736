"""Golden fixtures for the drop-in surface beyond the kernels, made by running the REFERENCE.

    python tests/golden/make_golden_dropin.py

Imports the reference in place from /root/reference/pkg/src (this container
only; numba's cache goes to a temp dir) and records, for the package-level
names the reference exports (pkg/src/twofold/__init__.py:11-42):
  - the LCG scalar API: next_raw / uniform01 / uniform_sym sequences and
    raw_to_uniform, per kind, dtype and seed (lcg.py:42-72);
  - fill() by its positional reference signature (sha256 + head);
  - Expansion / expansion_add / exact_sum / exact_dot components, including
    binary32 dots (exact products) and binary64 dots (rounded products)
    (expansion.py:73-126), and relative_error values;
  - the accuracy harness: run_accuracy_table(n=100000) rows and a small
    run_scaling_study (accuracy.py:73-173), whose seq flavor the GPU
    reproduces bit for bit.
Writes tests/golden/reference_dropin.json; the GPU box only reads it.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_ref_"))
sys.path.insert(0, REF)

import twofold as ref  # noqa: E402  (the reference)
from twofold import accuracy as ref_acc  # noqa: E402

DT = {"f32": np.float32, "f64": np.float64}


def h(v) -> str:
    return float(v).hex()


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    out = {"generator": f"tests/golden/make_golden_dropin.py (reference at {REF}, "
                        f"numba {__import__('numba').__version__}, numpy {np.__version__})"}

    # --- LCG scalar API ------------------------------------------------------
    scal = []
    for kind in ref.LcgKind:
        for seed in (0, 1, 12345, (1 << 40) + 7):
            g = ref.LcgState(kind, seed if kind is ref.LcgKind.MMIX else seed & 0xFFFFFFFF)
            raws = []
            for _ in range(6):
                r, g = ref.next_raw(g)
                raws.append(r)
            rec = {"kind": kind.value, "seed": seed, "raws": raws, "uniform01": {}, "uniform_sym": {}}
            for dt in ("f32", "f64"):
                g = ref.LcgState(kind, seed if kind is ref.LcgKind.MMIX else seed & 0xFFFFFFFF)
                u, s = [], []
                for _ in range(4):
                    v, g = ref.uniform01(g, DT[dt])
                    u.append(h(v))
                g = ref.LcgState(kind, seed if kind is ref.LcgKind.MMIX else seed & 0xFFFFFFFF)
                for _ in range(4):
                    v, g = ref.uniform_sym(g, DT[dt])
                    s.append(h(v))
                rec["uniform01"][dt] = u
                rec["uniform_sym"][dt] = s
            scal.append(rec)
    # the edge raws: 0 and 2^w - 1 (the latter rounds up to 1.0 at binary32)
    from twofold.lcg import raw_to_uniform
    edges = []
    for kind, w in ((ref.LcgKind.NUMERICAL_RECIPES, 32), (ref.LcgKind.MMIX, 64)):
        for raw in (0, 1, (1 << w) - 1, 1 << (w - 1)):
            for dt in ("f32", "f64"):
                for sym in (False, True):
                    edges.append({"kind": kind.value, "raw": raw, "dtype": dt, "sym": sym,
                                  "value": h(raw_to_uniform(raw, kind, DT[dt], sym))})
    out["lcg_scalar"] = scal
    out["lcg_edges"] = edges

    # --- fill() by the reference's positional signature ------------------------
    fills = []
    for kind in ref.LcgKind:
        for dt in ("f32", "f64"):
            for n, seed, sym in ((1, 1, False), (1000, 3, False), (100003, 7, True), (4097, 0, True)):
                a = ref.fill(kind, n, seed, DT[dt], sym)
                fills.append({"kind": kind.value, "n": n, "seed": seed, "dtype": dt, "sym": sym,
                              "sha256": sha(a), "head": [h(v) for v in a[:3]]})
    out["fill"] = fills

    # --- expansions -------------------------------------------------------------
    chains = []
    for vals in ([1.0, 2.0 ** -53, 2.0 ** -53], [1e100, 1.0, -1e100], [0.1] * 10, [1.0, -1.0],
                 [2.0 ** 1000, 2.0 ** -1000, -(2.0 ** 1000), 3.0]):
        e = ref.Expansion(())
        for v in vals:
            e = ref.expansion_add(e, v)
        chains.append({"values": [h(v) for v in vals], "components": [h(c) for c in e.components],
                       "float": h(float(e)), "hi": h(e.hi), "lo": h(e.lo), "is_zero": e.is_zero})
    out["expansion_add"] = chains

    exacts = []
    for dt in ("f32", "f64"):
        for n, seed in ((1, 1), (1000, 2), (65537, 3)):
            x = ref.fill(ref.LcgKind.MMIX, n, seed, DT[dt], True)
            y = ref.fill(ref.LcgKind.NUMERICAL_RECIPES, n, seed + 10, DT[dt], True)
            es = ref.exact_sum(x)
            ed = ref.exact_dot(x, y)
            exacts.append({"dtype": dt, "n": n, "seed": seed,
                           "sum": [h(c) for c in es.components], "dot": [h(c) for c in ed.components],
                           "rel_sum_direct": h(ref.relative_error(float(ref.sum_direct(x).value), es)),
                           "rel_dot_direct": h(ref.relative_error(float(ref.dot_direct(x, y).value), ed))})
    out["exact"] = exacts

    # --- the accuracy harness (seq flavor) ----------------------------------------
    rows = ref_acc.run_accuracy_table(n=100_000, seed=1)
    out["accuracy_table"] = {"n": 100_000, "seed": 1,
                             "rows": [{"precision": r.precision, "generator": r.generator, "interval": r.interval,
                                       "method": r.method, "rel_error": h(r.rel_error), "valid": r.valid}
                                      for r in rows]}
    st = ref_acc.run_scaling_study(ns=(1000, 10000), trials=5, seed=1)
    out["scaling_study"] = {"ns": [1000, 10000], "trials": 5, "seed": 1,
                            "rows": [{"n": r.n, "method": r.method, "median": h(r.median_abs_rel_error)}
                                     for r in st.rows],
                            "slopes": {k: (None if v is None else h(v)) for k, v in st.slopes.items()}}

    path = os.path.join(HERE, "reference_dropin.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print(f"wrote {path}")


if __name__ == "__main__":
    main()
