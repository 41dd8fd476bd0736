"""Exact (correctly rounded) sums and dot products on the GPU.

Device counterpart of the reference's expansion oracle (expansion.py):
``exact_sum`` / ``exact_dot`` return an ``ExactValue``, an ``Expansion``
(the reference's non-overlapping component tuple, increasing magnitude, so
``.components`` / ``.hi`` / ``.lo`` / ``float()`` / ``.add`` work as in
expansion.py:31-70) that also carries the device superaccumulator's exact
fixed-point limbs for rational checks.  Integer superaccumulation makes the
result independent of grid size and order.

Semantics follow expansion.py:112-126: ``exact_dot`` of binary32 data sums
the exact products (each f32*f32 product is exact in binary64); of binary64
data, the products rounded once to binary64.  ``rounded_products=True``
selects the binary32 kernels' own addends fl32(a*b) instead (what the
grid's error channel tracks), ``true_products=True`` the exact products at
either precision (what a TwoProduct dot tracks).
"""

from __future__ import annotations

import ctypes
import math
import threading
from dataclasses import dataclass
from fractions import Fraction

import torch

from . import _lib
from ._lib import check, lib
from .api import _as_tensor, _device_for, _dtype_code, _on_device, _stream_ptr

TF_EXACT_ABS = 1
TF_EXACT_TRUE_PRODUCTS = 2
_LIMBS = 72


def _two_sum(a: float, b: float) -> tuple[float, float]:
    """Knuth TwoSum on Python floats (binary64), for the host-side expansion
    bookkeeping of Expansion.add (the reference does the same in Python, eft.py:45-56)."""
    x = a + b
    bv = x - a
    av = x - bv
    return x, (a - av) + (b - bv)


@dataclass(frozen=True)
class Expansion:
    """Non-overlapping binary64 expansion, components in increasing magnitude
    (expansion.py:31-70); the zero expansion has no components."""

    components: tuple

    @property
    def is_zero(self) -> bool:
        return not self.components

    @property
    def hi(self) -> float:
        """Largest-magnitude component (0.0 for zero)."""
        return self.components[-1] if self.components else 0.0

    @property
    def lo(self) -> float:
        """Second-largest component (0.0 if absent)."""
        return self.components[-2] if len(self.components) > 1 else 0.0

    def __float__(self) -> float:
        return math.fsum(self.components)  # correctly rounded sum of the components

    def add(self, v: float) -> "Expansion":
        """Grow by one finite binary64 value, exactly (a TwoSum cascade)."""
        q = float(v)
        out = []
        for c in self.components:
            q, r = _two_sum(q, c)
            if r != 0.0:
                out.append(r)
        if q != 0.0:
            out.append(q)
        return Expansion(tuple(out))


ZERO = Expansion(())


def expansion_add(e: Expansion, v: float) -> Expansion:
    """Functional form of Expansion.add (expansion.py:73-75)."""
    return e.add(v)


def _components_of(q: Fraction) -> tuple:
    """Nearest-rounding decomposition of an exact rational into a non-overlapping
    binary64 expansion: c_top = fl(S), c_next = fl(S - c_top), ...  (|remainder|
    <= ulp/2 each step, so the components do not overlap); increasing magnitude."""
    comps = []
    while q != 0 and len(comps) < 64:
        try:
            c = float(q)  # correctly rounded (Fraction.__float__ rounds to nearest)
        except OverflowError:  # |S| beyond binary64: the reference's cascade overflows to inf too
            return (math.inf if q > 0 else -math.inf,)
        comps.append(c)
        q -= Fraction(c)
    return tuple(reversed(comps))


@dataclass(frozen=True)
class ExactValue(Expansion):
    """An Expansion computed on the device, plus its exact fixed-point limbs:
    S = sum limbs[k] 2^(32k-1074) + limbs[72] 2^(32*72-1074)."""

    limbs: tuple = ()

    def fraction(self) -> Fraction:
        v = sum(int(c) << (32 * k) for k, c in enumerate(self.limbs[:_LIMBS]))
        v += int(self.limbs[_LIMBS]) << (32 * _LIMBS)
        return Fraction(v, 1 << 1074)

    @classmethod
    def from_limbs(cls, limbs: tuple) -> "ExactValue":
        v = sum(int(c) << (32 * k) for k, c in enumerate(limbs[:_LIMBS])) + (int(limbs[_LIMBS]) << (32 * _LIMBS))
        return cls(_components_of(Fraction(v, 1 << 1074)), tuple(limbs))


class _Ws:
    def __init__(self):
        self._lock = threading.Lock()
        self._bufs = {}

    def get(self, dev: torch.device, nbytes: int):
        key = (dev.index, _stream_ptr(dev))
        with self._lock:
            rec = self._bufs.get(key)
            if rec is None or rec[0].numel() < nbytes:
                # both zero on the first call; every tf_exact leaves them zero
                rec = (torch.zeros(nbytes, dtype=torch.uint8, device=dev), torch.zeros(1, dtype=torch.int32, device=dev))
                self._bufs[key] = rec
            return rec


_ws = _Ws()


def _exact(x: torch.Tensor, y: torch.Tensor | None, flags: int) -> ExactValue:
    dev = _device_for(x)
    with torch.cuda.device(dev):
        x = _on_device(x, dev)
        y = _on_device(y, dev)
        _lib.ensure_canary(dev.index)
        recs, nbytes = ctypes.c_int64(0), ctypes.c_size_t(0)
        check(lib().tf_exact_workspace(ctypes.byref(recs), ctypes.byref(nbytes)), "tf_exact_workspace")
        buf, counter = _ws.get(dev, nbytes.value)
        out = torch.empty(2, dtype=torch.float64, device=dev)
        limbs = torch.empty(_LIMBS + 1, dtype=torch.int64, device=dev)
        check(lib().tf_exact(_dtype_code(x.dtype), x.data_ptr(), None if y is None else y.data_ptr(), x.numel(),
                             flags, out.data_ptr(), limbs.data_ptr(), buf.data_ptr(), nbytes.value,
                             counter.data_ptr(), _stream_ptr(dev)), "tf_exact")
    hi, lo = out.cpu().tolist()
    lt = tuple(limbs.cpu().tolist())
    if not math.isfinite(hi):  # a non-finite addend: the device reports inf / nan, the limbs hold the finite part
        return ExactValue((lo, hi) if lo != 0 else (hi,), lt)
    ev = ExactValue.from_limbs(lt)
    if math.isfinite(ev.hi) and (ev.hi, ev.lo) != (hi, lo):  # the device's own rounding of the limbs must agree
        raise RuntimeError(f"tf_exact: leading components ({hi!r}, {lo!r}) disagree with the limbs {ev.components!r}")
    return ev


def exact_sum(data, *, absolute: bool = False) -> ExactValue:
    """Exact sum of a float32/float64 array (expansion.exact_sum, expansion.py:104-109)."""
    x = _as_tensor(data)
    if x.numel() == 0:
        return ExactValue((), (0,) * (_LIMBS + 1))
    return _exact(x, None, TF_EXACT_ABS if absolute else 0)


def exact_dot(a, b, *, rounded_products: bool = False, true_products: bool = False,
              absolute: bool = False) -> ExactValue:
    """Exact sum of the elementwise products, as expansion.exact_dot (expansion.py:112-126):
    binary32 data -> the exact products; binary64 data -> the products rounded once
    to binary64 (the addends the binary64 dot kernels see).

    rounded_products=True: the products rounded in the DATA precision for either
    dtype — for binary32 the addends fl32(a*b) the binary32 dot kernels sum, so
    the grid's error channel is judged against its own addends.
    true_products=True: the exact products for either dtype (the TwoProduct target).
    """
    if rounded_products and true_products:
        raise ValueError("rounded_products and true_products are exclusive")
    x, y = _as_tensor(a), _as_tensor(b)
    if x.dtype != y.dtype:
        raise TypeError("dot operands must share a dtype")
    if x.shape != y.shape:
        raise ValueError("exact_dot needs equal-length arrays")
    if x.numel() == 0:
        return ExactValue((), (0,) * (_LIMBS + 1))
    exact_products = true_products or (x.dtype == torch.float32 and not rounded_products)
    flags = (TF_EXACT_TRUE_PRODUCTS if exact_products else 0) | (TF_EXACT_ABS if absolute else 0)
    return _exact(x, y, flags)


def relative_error(approx: float, reference: Expansion) -> float:
    """(approx - reference) / reference from the two leading components,
    exactly as expansion.relative_error (expansion.py:129-140)."""
    if reference.is_zero:
        raise ValueError("relative error against a zero reference is undefined")
    hi, lo = reference.hi, reference.lo
    return ((float(approx) - hi) - lo) / (hi + lo)


__all__ = ["Expansion", "ExactValue", "ZERO", "expansion_add", "exact_sum", "exact_dot", "relative_error"]
