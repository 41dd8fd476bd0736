"""The reference's LCG data API (pkg/src/twofold/lcg.py) with the array fill on the GPU.

Scalar side (``LcgKind``, ``LcgState``, ``next_raw``, ``raw_to_uniform``,
``uniform01``, ``uniform_sym``): immutable generator states advanced with
Python integers — the reference's own semantics (lcg.py:20-72), host logic
like its scalar API.  ``fill`` is the array side: the recurrence runs on the
device with jump-ahead (tf_lcg_fill, csrc/misc.cu; s_i = a^i s_0 + c (a^i - 1)
/ (a - 1) mod 2^w per thread block), bit-identical to the reference's numba
fill (lcg.py:75-116; tests/test_gpu_dropin.py compares sha256 of the bytes
with the reference-generated goldens).  ``fill`` returns a numpy array like
the reference, or a CUDA tensor when ``device`` is given.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

import numpy as np
import torch


class LcgKind(Enum):
    """lcg.py:20-22: the 32-bit Numerical Recipes and Knuth's 64-bit MMIX generators."""

    NUMERICAL_RECIPES = "nr"
    MMIX = "mmix"


# width, multiplier, increment (lcg.py:26-29)
_WIDTH = {LcgKind.NUMERICAL_RECIPES: 32, LcgKind.MMIX: 64}
_MUL = {LcgKind.NUMERICAL_RECIPES: 1664525, LcgKind.MMIX: 6364136223846793005}
_INC = {LcgKind.NUMERICAL_RECIPES: 1013904223, LcgKind.MMIX: 1442695040888963407}

DEFAULT_SEED = 1


@dataclass(frozen=True)
class LcgState:
    """Immutable generator state (lcg.py:34-39); advancing returns a new state."""

    kind: LcgKind
    state: int = DEFAULT_SEED


def next_raw(g: LcgState) -> tuple[int, LcgState]:
    """One step s' = (a*s + c) mod 2^width; returns (s', new state) (lcg.py:42-46)."""
    mask = (1 << _WIDTH[g.kind]) - 1
    s = (_MUL[g.kind] * g.state + _INC[g.kind]) & mask
    return s, LcgState(g.kind, s)


def raw_to_uniform(raw: int, kind: LcgKind, dtype=np.float64, sym: bool = False):
    """raw / 2^width rounded once to `dtype` ([0,1)), or 2u - 1 in `dtype` when sym
    (lcg.py:49-60; note the reference's "[0,1)" can round up to exactly 1.0)."""
    t = np.dtype(dtype).type
    u = t(raw) / t(2.0 ** _WIDTH[kind])
    return t(2) * u - t(1) if sym else u


def uniform01(g: LcgState, dtype=np.float64):
    """One draw in [0,1): (value, new state) (lcg.py:63-66)."""
    raw, nxt = next_raw(g)
    return raw_to_uniform(raw, g.kind, dtype), nxt


def uniform_sym(g: LcgState, dtype=np.float64):
    """One draw in [-1,1): (value, new state) (lcg.py:69-72)."""
    raw, nxt = next_raw(g)
    return raw_to_uniform(raw, g.kind, dtype, sym=True), nxt


def _kind(kind) -> LcgKind:
    if isinstance(kind, LcgKind):
        return kind
    try:
        return LcgKind(kind)
    except ValueError:
        raise ValueError(f"unknown LCG kind {kind!r}") from None


def fill(kind, n: int, seed: int = DEFAULT_SEED, dtype=np.float64, sym: bool = False, *,
         device=None):
    """n draws of the generator from `seed` (lcg.py:108-116), generated on the GPU.

    Returns a numpy array of `dtype` (the reference's result type) unless
    `device` is given, in which case the CUDA tensor stays on that device.
    """
    from .gen import lcg_fill
    k = _kind(kind)
    tdt = torch.float32 if np.dtype(dtype) == np.float32 else torch.float64
    if np.dtype(dtype) not in (np.float32, np.float64):
        raise TypeError(f"unsupported dtype {np.dtype(dtype)}; use float32/float64")
    if n < 0:
        raise ValueError("negative length")
    if device is not None:
        return lcg_fill(k.value, n, seed, tdt, sym, device=device)
    if n == 0:
        return np.empty(0, dtype)
    return lcg_fill(k.value, n, seed, tdt, sym).cpu().numpy()


__all__ = ["LcgKind", "LcgState", "DEFAULT_SEED", "next_raw", "raw_to_uniform", "uniform01", "uniform_sym",
           "fill"]
