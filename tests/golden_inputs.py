"""Rebuild the golden fixtures' inputs from their specs (oracle restatements)."""

import hashlib

import numpy as np

DT = {"f32": np.float32, "f64": np.float64}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def make(O, spec):
    if spec is None:
        return None
    dt = DT[spec["dtype"]]
    kind = spec["kind"]
    if kind == "lcg":
        return O.lcg_fill(spec["lcg"], spec["n"], spec["seed"], dt, spec["sym"])
    if kind == "philox":
        return O.philox_fill(spec["dist"], spec["n"], spec["seed"], spec["stream"], spec.get("offset", 0), dt,
                             total=spec.get("total", 0))
    if kind == "literal":
        return np.array([float.fromhex(v) for v in spec["values"]], dt)
    if kind == "arange":
        return np.arange(1, spec["n"] + 1, dtype=dt)
    raise ValueError(kind)


def load_inputs(O, golden, section=None):
    out = {}
    recs = golden["inputs"] if section is None else golden[section]["inputs"]
    for name, rec in recs.items():
        x = make(O, rec["x"])
        y = make(O, rec["y"])
        out[name] = (x, y)
    return out
