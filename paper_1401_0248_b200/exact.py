"""Exact (correctly rounded) sums and dot products on the GPU.

Device counterpart of the reference's expansion oracle (expansion.py:79-140):
``exact_sum`` / ``exact_dot`` return the exact value's two leading binary64
components (hi = fl(S), lo = fl(S - hi)) — exactly what the reference's
``relative_error`` consumes (``Expansion.hi`` / ``.lo``) — plus the full
fixed-point representation for rational checks.  Integer superaccumulation
makes the result independent of grid size and order.
"""

from __future__ import annotations

import ctypes
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


@dataclass(frozen=True)
class ExactValue:
    """hi = fl(S), lo = fl(S - hi); limbs: S = sum limbs[k] 2^(32k-1074) + limbs[72] 2^(32*72-1074)."""

    hi: float
    lo: float
    limbs: tuple

    def fraction(self) -> Fraction:
        v = sum(int(c) << (32 * k) for k, c in enumerate(self.limbs[:_LIMBS]))
        v += int(self.limbs[_LIMBS]) << (32 * _LIMBS)
        return Fraction(v, 1 << 1074)

    @property
    def is_zero(self) -> bool:
        return self.hi == 0.0

    def __float__(self) -> float:
        return self.hi


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
    return ExactValue(hi, lo, tuple(limbs.cpu().tolist()))


def exact_sum(data, *, absolute: bool = False) -> ExactValue:
    """Exact sum of a float32/float64 array (expansion.exact_sum, expansion.py:104-109)."""
    x = _as_tensor(data)
    if x.numel() == 0:
        return ExactValue(0.0, 0.0, (0,) * (_LIMBS + 1))
    return _exact(x, None, TF_EXACT_ABS if absolute else 0)


def exact_dot(a, b, *, true_products: bool = False, absolute: bool = False) -> ExactValue:
    """Exact sum of the products.  Default: the products rounded in the data
    precision — the identical addends the twofold dot kernels sum (for binary64
    this is expansion.exact_dot, expansion.py:112-126).  true_products=True:
    the exact products (what a TwoProduct dot tracks; for binary32 this is the
    reference's exact_dot)."""
    x, y = _as_tensor(a), _as_tensor(b)
    if x.dtype != y.dtype:
        raise TypeError("dot operands must share a dtype")
    if x.shape != y.shape:
        raise ValueError("exact_dot needs equal-length arrays")
    if x.numel() == 0:
        return ExactValue(0.0, 0.0, (0,) * (_LIMBS + 1))
    flags = (TF_EXACT_TRUE_PRODUCTS if true_products else 0) | (TF_EXACT_ABS if absolute else 0)
    return _exact(x, y, flags)


def relative_error(approx: float, reference: ExactValue) -> float:
    """(approx - reference) / reference from the two leading components,
    exactly as expansion.relative_error (expansion.py:129-140)."""
    if reference.is_zero:
        raise ValueError("relative error against a zero reference is undefined")
    hi, lo = reference.hi, reference.lo
    return ((float(approx) - hi) - lo) / (hi + lo)


__all__ = ["ExactValue", "exact_sum", "exact_dot", "relative_error"]
