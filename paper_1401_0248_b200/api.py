"""Drop-in mirror of the reference's kernel API on B200 kernels.

Reference surface (pkg/src/twofold): ``Method`` (kernels.py:44-49),
``Flavor`` (:57-104), ``SumResult`` (:107-120), ``Twofold`` (eft.py:21-25),
``run_flavor`` (kernels.py:591-640), the ten wrappers (:669-706),
``raw_sum_kernel`` (:651-661), ``fast_two_sum`` / ``two_sum`` /
``rounding_canary`` (eft.py:28-66).  Same names, argument meaning, result
types and exceptions.  Every flavor runs on the GPU:

  ``cuda``          the grid reduction: per-thread recurrences + deterministic
                    TwoSum trees, HBM-bandwidth bound; value+error tracks the
                    exact sum like any non-sequential flavor
  ``seq``           one GPU thread running the reference recurrence left to right:
                    bit-identical to the reference's sequential kernels (the
                    default of the ten sum_* / dot_* wrappers, as in the reference)
  ``unroll:k/vec:k`` k GPU lanes with the reference's lane merge: bit-identical
                    to the reference's lane kernels

The ten wrappers run ``default_flavor()``: ``seq`` unless changed with
``set_default_flavor`` / ``using_flavor`` or the environment variable
``TWOFOLD_B200_FLAVOR`` (e.g. ``cuda``), so ``import paper_1401_0248_b200 as
twofold`` returns the reference's bits until the caller opts into the grid;
each wrapper also takes an explicit ``flavor=`` keyword.

Inputs may be numpy arrays / array-likes (copied to the GPU; large host
arrays are streamed in leaf-aligned chunks overlapped with the reduction) or
torch tensors (CUDA tensors are reduced in place).  There is no CPU
fallback: without the CUDA library or a GPU every compute call raises.
"""

from __future__ import annotations

import contextlib
import ctypes
import functools
import threading
from dataclasses import dataclass
from enum import Enum
from typing import NamedTuple

import numpy as np
import torch

from . import _lib
from ._lib import check, lib


class Method(Enum):
    DIRECT = "direct"
    WIDE = "wide"
    TWOFOLD_FAST = "twofold-fast"
    TWOFOLD_RIGOROUS = "twofold-rigorous"
    KAHAN = "kahan"


_METHOD_ID = {Method.DIRECT: 0, Method.WIDE: 1, Method.TWOFOLD_FAST: 2,
              Method.TWOFOLD_RIGOROUS: 3, Method.KAHAN: 4}
TRACK_PRODUCT = 0x100  # TF_TRACK_PRODUCT: opt-in TwoProduct dots (include/twofold_b200.h)


def _mid(method: Method, track_product: bool = False, dot: bool = True) -> int:
    """C-ABI method id; track_product adds the exact product round-off to the
    error channel (Dot2-style; the reference tracks summation round-off only,
    kernels.py:23-26), valid for twofold dot products."""
    if not track_product:
        return _METHOD_ID[method]
    if method not in (Method.TWOFOLD_FAST, Method.TWOFOLD_RIGOROUS):
        raise ValueError("track_product needs a twofold method")
    if not dot:
        raise ValueError("track_product applies to dot products")
    return _METHOD_ID[method] | TRACK_PRODUCT
_TWOFOLD_METHODS = (Method.TWOFOLD_FAST, Method.TWOFOLD_RIGOROUS)

_LANE_RANGE = (2, 16)
# One SIMD register's worth of lanes per precision (kernels.py:52-54).
_DEFAULT_LANES = {np.dtype(np.float32): 8, np.dtype(np.float64): 4}

_KINDS = ("seq", "unroll", "vec", "cuda")


@dataclass(frozen=True)
class Flavor:
    """Execution flavor; lanes == 0 means "default for the precision".

    Kinds are the reference's "seq" | "unroll" | "vec" (kernels.py:57-104)
    plus "cuda", the grid reduction.  Validation and parsing follow the
    reference exactly; "cuda" takes no lane count.
    """

    kind: str
    lanes: int = 0

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ValueError(f"unknown flavor kind {self.kind!r}")
        if self.kind in ("seq", "cuda"):
            if self.lanes:
                raise ValueError(f"{'sequential' if self.kind == 'seq' else 'cuda'} flavor takes no lane count")
        elif self.lanes:
            lo, hi = _LANE_RANGE
            if not (lo <= self.lanes <= hi) or self.lanes & (self.lanes - 1):
                raise ValueError(f"lane count must be a power of two in [{lo}, {hi}]")

    @classmethod
    def sequential(cls) -> "Flavor":
        return cls("seq")

    @classmethod
    def unrolled(cls, k: int = 0) -> "Flavor":
        return cls("unroll", k)

    @classmethod
    def vectorized(cls, w: int = 0) -> "Flavor":
        return cls("vec", w)

    @classmethod
    def cuda(cls) -> "Flavor":
        return cls("cuda")

    @classmethod
    def parse(cls, text: str) -> "Flavor":
        """Parse "seq", "unroll[:k]", "vec[:w]" or "cuda" (CLI syntax)."""
        name, _, arg = text.partition(":")
        lanes = int(arg) if arg else 0
        if name == "seq":
            return cls.sequential()
        if name == "unroll":
            return cls.unrolled(lanes)
        if name == "vec":
            return cls.vectorized(lanes)
        if name == "cuda":
            return cls("cuda", lanes)
        raise ValueError(f"unknown flavor {text!r}; valid: seq, unroll:k, vec:w, cuda")

    def __str__(self) -> str:
        if self.kind in ("seq", "cuda"):
            return self.kind
        return f"{self.kind}:{self.lanes}" if self.lanes else self.kind


class Twofold(NamedTuple):
    """Value + error pair approximating one real number (eft.py:21-25)."""

    value: float
    error: float


@dataclass(frozen=True)
class SumResult:
    """Kernel output: twofold sum plus the attributed addition count."""

    twofold: Twofold
    adds_performed: int

    @property
    def value(self):
        return self.twofold.value

    @property
    def error(self):
        return self.twofold.error


@dataclass(frozen=True)
class RowsResult:
    """Batched row-wise output: device tensors of per-row values and errors."""

    values: torch.Tensor
    errors: torch.Tensor
    adds_performed: int  # per row (= cols), by the one-add-per-element convention


_CUDA = Flavor.cuda()
_SEQ = Flavor.sequential()


def _env_flavor() -> Flavor:
    import os
    spec = os.environ.get("TWOFOLD_B200_FLAVOR", "").strip()
    return Flavor.parse(spec) if spec else _SEQ


_default_flavor = [_env_flavor()]


def default_flavor() -> Flavor:
    """The flavor the ten sum_* / dot_* wrappers run (process-wide)."""
    return _default_flavor[0]


def set_default_flavor(flavor) -> Flavor:
    """Set the wrappers' flavor (a Flavor or its CLI text, e.g. "cuda"); returns the previous one.
    The reference's wrappers are sequential (kernels.py:666-706); "cuda" trades those
    exact bits for the grid reduction's HBM-bound speed and tree accuracy."""
    fl = Flavor.parse(flavor) if isinstance(flavor, str) else flavor
    if not isinstance(fl, Flavor):
        raise TypeError("flavor must be a Flavor or a flavor string")
    prev, _default_flavor[0] = _default_flavor[0], fl
    return prev


@contextlib.contextmanager
def using_flavor(flavor):
    """Context manager form of set_default_flavor (restores the previous flavor)."""
    prev = set_default_flavor(flavor)
    try:
        yield default_flavor()
    finally:
        set_default_flavor(prev)

# ---------------------------------------------------------------------------
# Input handling (kernels.py:574-584 semantics).

_TORCH_OK = (torch.float32, torch.float64)


def _as_tensor(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        t = a
    else:
        arr = np.ascontiguousarray(a)
        if arr.dtype not in (np.float32, np.float64):
            raise TypeError(f"unsupported dtype {arr.dtype}; use float32/float64")
        t = torch.from_numpy(arr)
    if t.dtype not in _TORCH_OK:
        raise TypeError(f"unsupported dtype {t.dtype}; use float32/float64")
    if t.dim() != 1:
        raise ValueError(f"expected a 1-D array, got shape {tuple(t.shape)}")
    return t


def _check_input(data, b):
    x = _as_tensor(data)
    y = None
    if b is not None:
        y = _as_tensor(b)
        if y.dtype != x.dtype:
            raise TypeError("dot operands must share a dtype")
        if y.shape != x.shape:
            raise ValueError("dot operands must have equal length")
    return x, y


def _dtype_code(t: torch.dtype) -> int:
    return _lib.TF_F32 if t == torch.float32 else _lib.TF_F64


def _np_type(t: torch.dtype):
    return np.float32 if t == torch.float32 else np.float64


def _acc_dtype(method: Method, t: torch.dtype) -> torch.dtype:
    return torch.float64 if method is Method.WIDE else t


def _device_for(x: torch.Tensor) -> torch.device:
    if x.is_cuda:
        return x.device
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device available: the twofold B200 library has no CPU path")
    return torch.device("cuda", torch.cuda.current_device())


def _on_device(t: torch.Tensor | None, dev: torch.device) -> torch.Tensor | None:
    if t is None:
        return None
    if t.is_cuda:
        if t.device != dev:
            raise ValueError(f"operands live on different devices ({t.device} vs {dev})")
        return t.contiguous()
    return t.to(dev, non_blocking=t.is_pinned()).contiguous()


def _ptr(t: torch.Tensor | None):
    return None if t is None else t.data_ptr()


def _stream_ptr(dev: torch.device) -> int:
    return torch.cuda.current_stream(dev).cuda_stream


def _on(dev: torch.device):
    """torch.cuda.device(dev), skipped when dev is already current (saves µs per call)."""
    if dev.index == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(dev)


# ---------------------------------------------------------------------------
# Per-(device, stream) scratch: grow-only partials + zeroed retire counters
# (the kernels leave counters zero, so one buffer serves every call on a stream).

class _Scratch:
    def __init__(self):
        self._lock = threading.Lock()
        self._bufs: dict[tuple[int, int], list] = {}

    def get(self, dev: torch.device, partials_bytes: int, counters: int, stream_ptr: int | None = None):
        key = (dev.index, _stream_ptr(dev) if stream_ptr is None else stream_ptr)
        rec = self._bufs.get(key)
        if rec is not None and rec[0].numel() >= partials_bytes and rec[1].numel() >= counters:
            return rec[0], rec[1]
        with self._lock:
            rec = self._bufs.get(key)
            if rec is None:
                rec = [torch.empty(0, dtype=torch.uint8, device=dev),
                       torch.zeros(0, dtype=torch.int32, device=dev)]
                self._bufs[key] = rec
            if rec[0].numel() < partials_bytes:
                rec[0] = torch.empty(max(partials_bytes, 2 * rec[0].numel()), dtype=torch.uint8, device=dev)
            if rec[1].numel() < counters:
                rec[1] = torch.zeros(max(counters, 2 * rec[1].numel(), 64), dtype=torch.int32, device=dev)
            return rec[0], rec[1]


_scratch = _Scratch()


def workspace_size(method: Method, dtype: torch.dtype, rows: int, cols: int, leaf_log2: int = 0):
    """(partials bytes, counters, leaves per row) — a pure function, cached."""
    return _workspace_size(_METHOD_ID[method], _dtype_code(dtype), rows, cols, leaf_log2)


@functools.lru_cache(maxsize=4096)
def _workspace_size(mid: int, dcode: int, rows: int, cols: int, leaf_log2: int):
    pb = ctypes.c_size_t(0)
    cnt = ctypes.c_int64(0)
    leaves = ctypes.c_int64(0)
    check(lib().tf_workspace_size(mid, dcode, rows, cols, leaf_log2, pb, cnt, leaves), "tf_workspace_size")
    return pb.value, cnt.value, leaves.value


def leaf_log2_for(dtype: torch.dtype, n: int) -> int:
    """Auto leaf size of the grid flavor (a pure function of dtype and n)."""
    return int(lib().tf_leaf_log2(_dtype_code(dtype), n))


# ---------------------------------------------------------------------------
# Device-side launchers (asynchronous; return device pairs).

def _reduce_grid(method: Method, x: torch.Tensor, y: torch.Tensor | None, leaf_log2: int = 0,
                 out: torch.Tensor | None = None, track_product: bool = False) -> torch.Tensor:
    dev = x.device
    _lib.ensure_canary(dev.index)
    acc = _acc_dtype(method, x.dtype)
    if out is None:
        out = torch.empty(2, dtype=acc, device=dev)
    n = x.numel()
    pb, cnt, _ = workspace_size(method, x.dtype, 1, n, leaf_log2)
    sp = _stream_ptr(dev)
    parts, ctrs = _scratch.get(dev, pb, cnt, sp)  # cached per stream; also feeds leaf splitting
    rc = lib().tf_reduce(_mid(method, track_product, y is not None), _dtype_code(x.dtype), x.data_ptr(), _ptr(y), n,
                         leaf_log2, out.data_ptr(), parts.data_ptr(), pb, ctrs.data_ptr(), cnt, sp)
    if rc:
        check(rc, "tf_reduce")
    return out


def merge_pairs(method: Method, pairs: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Balanced TwoSum/Kahan/plain tree over a (k, 2) device tensor of pairs."""
    pairs = pairs.contiguous()
    dev = pairs.device
    with torch.cuda.device(dev):
        if out is None:
            out = torch.empty(2, dtype=pairs.dtype, device=dev)
        data_dtype = torch.float32 if (pairs.dtype == torch.float32) else torch.float64
        if method is Method.WIDE:
            data_dtype = torch.float32
        check(lib().tf_merge_tree(_METHOD_ID[method], _dtype_code(data_dtype), pairs.data_ptr(),
                                  pairs.numel() // 2, out.data_ptr(), _stream_ptr(dev)), "tf_merge_tree")
        return out


def _host_pair(method: Method, x: torch.Tensor, y: torch.Tensor | None, dev: torch.device,
               leaf_log2: int = 0, track_product: bool = False, engine=None) -> np.ndarray:
    """Blocking grid flavor through the native host-buffer engine
    (tf_host_reduce, csrc/host.cu).  Host tensors: pinned staging, leaf-aligned
    chunks whose copies overlap the leaf kernels; CUDA tensors (of `dev`):
    reduced in place after the current stream's pending work, the pair stored
    straight into mapped host memory.  Bit-identical to the device path.
    Returns the raw (value, error) pair as a numpy array."""
    _lib.ensure_canary(dev.index)
    x = x.contiguous()
    y = None if y is None else y.contiguous()
    pair = np.empty(2, dtype=_np_type(_acc_dtype(method, x.dtype)))
    eng = engine if engine is not None else _lib.host_engine(dev.index)
    check(lib().tf_host_reduce(eng, _mid(method, track_product, y is not None), _dtype_code(x.dtype),
                               x.data_ptr(), None if y is None else y.data_ptr(), x.numel(), leaf_log2,
                               pair.ctypes.data, _stream_ptr(dev)), "tf_host_reduce")
    return pair


def _reduce_host(method: Method, x: torch.Tensor, y: torch.Tensor | None, dev: torch.device,
                 leaf_log2: int = 0, out: torch.Tensor | None = None, track_product: bool = False) -> torch.Tensor:
    """_host_pair, delivered as a 2-element device tensor (reduce()'s result form)."""
    pair = torch.from_numpy(_host_pair(method, x, y, dev, leaf_log2, track_product))
    if out is None:
        return pair.to(dev)
    return out.copy_(pair)


def _reduce_seq(method: Method, x, y, dev, track_product: bool = False) -> torch.Tensor:
    _lib.ensure_canary(dev.index)
    out = torch.empty(2, dtype=_acc_dtype(method, x.dtype), device=dev)
    check(lib().tf_reduce_seq(_mid(method, track_product, y is not None), _dtype_code(x.dtype), _ptr(x), _ptr(y), x.numel(),
                              out.data_ptr(), _stream_ptr(dev)), "tf_reduce_seq")
    return out


def _reduce_lanes(method: Method, x, y, k: int, dev, track_product: bool = False) -> torch.Tensor:
    _lib.ensure_canary(dev.index)
    out = torch.empty(2, dtype=_acc_dtype(method, x.dtype), device=dev)
    check(lib().tf_reduce_lanes(_mid(method, track_product, y is not None), _dtype_code(x.dtype), _ptr(x), _ptr(y), x.numel(), k,
                                out.data_ptr(), _stream_ptr(dev)), "tf_reduce_lanes")
    return out


def reduce(method: Method, data, b=None, *, flavor: Flavor = _CUDA, leaf_log2: int = 0,
           out: torch.Tensor | None = None, track_product: bool = False) -> torch.Tensor:
    """Asynchronous form of run_flavor: returns the raw (value, error) pair as a
    2-element device tensor without synchronizing (for KAHAN the error slot
    holds the pending compensation).  Inputs must already be CUDA tensors for
    the result to stay asynchronous.  track_product: opt-in TwoProduct dot."""
    x, y = _check_input(data, b)
    if method is Method.WIDE and x.dtype != torch.float32:
        raise TypeError("wide accumulation is defined for float32 data only")
    _mid(method, track_product, y is not None)  # validate before touching the device
    dev = _device_for(x)
    with _on(dev):  # the C library launches on the current device
        if flavor.kind == "cuda":
            if _all_host(x, y):
                return _reduce_host(method, x, y, dev, leaf_log2, out, track_product)
            return _reduce_grid(method, _on_device(x, dev), _on_device(y, dev), leaf_log2, out, track_product)
        xd, yd = _on_device(x, dev), _on_device(y, dev)
        if flavor.kind == "seq":
            return _reduce_seq(method, xd, yd, dev, track_product)
        k = flavor.lanes or _DEFAULT_LANES[np.dtype(_np_type(x.dtype))]
        return _reduce_lanes(method, xd, yd, k, dev, track_product)


def _all_host(x: torch.Tensor, y: torch.Tensor | None) -> bool:
    return not x.is_cuda and (y is None or not y.is_cuda)


def _finish(method: Method, pair, dtype: torch.dtype, n: int) -> SumResult:
    v, e = (pair.cpu() if torch.is_tensor(pair) else pair).tolist()
    t = np.float64 if method is Method.WIDE else _np_type(dtype)
    if method in _TWOFOLD_METHODS:
        return SumResult(Twofold(t(v), t(e)), n)
    return SumResult(Twofold(t(v), t(0)), n)


def run_flavor(method: Method, flavor: Flavor, data, b=None, *, track_product: bool = False) -> SumResult:
    """Run one method in one flavor over data (dot product when b is given).

    Mirrors kernels.py:591-640: same validation order and exceptions, result
    fields typed like the data (np.float64 for wide), error 0 for
    non-twofold methods, adds_performed == len(data).  Non-sequential flavors
    ("cuda", "unroll", "vec") associate differently from "seq" and are not
    bitwise reproductions of it; they satisfy the same accuracy contracts.
    """
    if flavor.kind == "cuda" and type(data) is np.ndarray and (b is None or type(b) is np.ndarray):
        return _run_numpy(method, data, b, track_product)
    x, y = _check_input(data, b)
    n = x.numel()
    if method is Method.WIDE and x.dtype != torch.float32:
        raise TypeError("wide accumulation is defined for float32 data only")
    if method not in _METHOD_ID:
        raise ValueError(f"unknown method {method!r}")
    if flavor.kind == "cuda" and (_all_host(x, y) or (x.is_cuda and (y is None or y.device == x.device))):
        # one blocking native call (host or same-device operands)
        _mid(method, track_product, y is not None)
        pair = _host_pair(method, x, y, _device_for(x), track_product=track_product)
    else:
        pair = reduce(method, x, y, flavor=flavor, track_product=track_product)
    return _finish(method, pair, x.dtype, n)


_NP_CODE = {np.dtype(np.float32): _lib.TF_F32, np.dtype(np.float64): _lib.TF_F64}


def _run_numpy(method: Method, a: np.ndarray, b: np.ndarray | None, track_product: bool) -> SumResult:
    """run_flavor(method, "cuda", a[, b]) for numpy arrays: the same checks and
    result as the general path, minus the torch round trip — host pointers go
    straight to the native host-buffer engine (tf_host_reduce)."""
    code = _NP_CODE.get(a.dtype)
    if code is None:
        raise TypeError(f"unsupported dtype {a.dtype}; use float32/float64")
    if a.ndim != 1:
        raise ValueError(f"expected a 1-D array, got shape {a.shape}")
    if b is not None:
        if _NP_CODE.get(b.dtype) is None:
            raise TypeError(f"unsupported dtype {b.dtype}; use float32/float64")
        if b.ndim != 1:
            raise ValueError(f"expected a 1-D array, got shape {b.shape}")
        if b.dtype != a.dtype:
            raise TypeError("dot operands must share a dtype")
        if b.shape != a.shape:
            raise ValueError("dot operands must have equal length")
    if method is Method.WIDE and code != _lib.TF_F32:
        raise TypeError("wide accumulation is defined for float32 data only")
    if method not in _METHOD_ID:
        raise ValueError(f"unknown method {method!r}")
    mid = _mid(method, track_product, b is not None)
    if not a.flags.c_contiguous:
        a = np.ascontiguousarray(a)
    if b is not None and not b.flags.c_contiguous:
        b = np.ascontiguousarray(b)
    global _cuda_seen
    if not _cuda_seen:
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device available: the twofold B200 library has no CPU path")
        _cuda_seen = True
    dev = torch.cuda.current_device()
    _lib.ensure_canary(dev)
    pair, pair_ptr = _pair_buffer(np.float64 if method is Method.WIDE else a.dtype)
    rc = lib().tf_host_reduce(_lib.host_engine(dev), mid, code, a.__array_interface__["data"][0],
                              None if b is None else b.__array_interface__["data"][0], a.shape[0], 0, pair_ptr,
                              None)
    if rc:
        check(rc, "tf_host_reduce")
    if method in _TWOFOLD_METHODS:
        return SumResult(Twofold(pair[0], pair[1]), a.shape[0])  # numpy scalars: copies, the buffer is reused
    return SumResult(Twofold(pair[0], pair.dtype.type(0)), a.shape[0])


_cuda_seen = False
_pair_tls = threading.local()


def _pair_buffer(dtype) -> tuple[np.ndarray, int]:
    """A per-thread 2-element result buffer and its address (one per dtype)."""
    cache = getattr(_pair_tls, "bufs", None)
    if cache is None:
        cache = _pair_tls.bufs = {}
    rec = cache.get(dtype)
    if rec is None:
        buf = np.empty(2, dtype=dtype)
        rec = cache[dtype] = (buf, buf.ctypes.data)
    return rec


def raw_sum_kernel(method: Method, flavor: Flavor, dtype):
    """The device launcher itself, plus whether it returns a pair (kernels.py:651-661).

    The returned callable takes a CUDA tensor and returns the raw 2-element
    device pair without synchronizing — the analogue of driving the compiled
    kernel from inside a timing loop (or a CUDA graph)."""
    tdt = torch.float32 if np.dtype(dtype) == np.float32 else torch.float64

    def kern(data: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if data.dtype != tdt:
            raise TypeError("data dtype does not match the kernel's")
        return reduce(method, data, flavor=flavor, out=out)

    return kern, method in _TWOFOLD_METHODS


def _fl(flavor) -> Flavor:
    if flavor is None:
        return _default_flavor[0]
    return Flavor.parse(flavor) if isinstance(flavor, str) else flavor


# The ten reference wrappers (kernels.py:666-706): default_flavor(), i.e. the
# reference's sequential bits unless the caller opts into the grid.

def sum_direct(data, *, flavor=None) -> SumResult:
    return run_flavor(Method.DIRECT, _fl(flavor), data)


def sum_wide(data, *, flavor=None) -> SumResult:
    return run_flavor(Method.WIDE, _fl(flavor), data)


def sum_twofold_fast(data, *, flavor=None) -> SumResult:
    return run_flavor(Method.TWOFOLD_FAST, _fl(flavor), data)


def sum_twofold_rigorous(data, *, flavor=None) -> SumResult:
    return run_flavor(Method.TWOFOLD_RIGOROUS, _fl(flavor), data)


def sum_kahan(data, *, flavor=None) -> SumResult:
    return run_flavor(Method.KAHAN, _fl(flavor), data)


def dot_direct(a, b, *, flavor=None) -> SumResult:
    return run_flavor(Method.DIRECT, _fl(flavor), a, b)


def dot_wide(a, b, *, flavor=None) -> SumResult:
    return run_flavor(Method.WIDE, _fl(flavor), a, b)


def dot_twofold_fast(a, b, *, flavor=None, track_product: bool = False) -> SumResult:
    return run_flavor(Method.TWOFOLD_FAST, _fl(flavor), a, b, track_product=track_product)


def dot_twofold_rigorous(a, b, *, flavor=None, track_product: bool = False) -> SumResult:
    return run_flavor(Method.TWOFOLD_RIGOROUS, _fl(flavor), a, b, track_product=track_product)


def dot_kahan(a, b, *, flavor=None) -> SumResult:
    return run_flavor(Method.KAHAN, _fl(flavor), a, b)


# ---------------------------------------------------------------------------
# Batched row-wise family (no reference analogue).

def _as_rows(a) -> torch.Tensor:
    t = a if isinstance(a, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(a))
    if t.dtype not in _TORCH_OK:
        raise TypeError(f"unsupported dtype {t.dtype}; use float32/float64")
    if t.dim() != 2:
        raise ValueError(f"expected a 2-D (rows, cols) array, got shape {tuple(t.shape)}")
    if t.stride(1) != 1:
        t = t.contiguous()
    return t


def reduce_rows(method: Method, X, Y=None, *, leaf_log2: int = 0,
                out: torch.Tensor | None = None, track_product: bool = False) -> torch.Tensor:
    """Asynchronous row-wise reduction: returns a (rows, 2) device tensor of raw pairs.
    Row r is bit-identical to reduce(method, X[r], Y[r]) with the same leaf size."""
    x = _as_rows(X)
    y = None if Y is None else _as_rows(Y)
    if y is not None:
        if y.dtype != x.dtype:
            raise TypeError("dot operands must share a dtype")
        if y.shape != x.shape:
            raise ValueError("dot operands must have equal shapes")
    if method is Method.WIDE and x.dtype != torch.float32:
        raise TypeError("wide accumulation is defined for float32 data only")
    mid = _mid(method, track_product, y is not None)
    dev = _device_for(x)
    with torch.cuda.device(dev):
        if _all_host(x, y):  # host matrices: the host-buffer engine, row blocks overlapped
            _lib.ensure_canary(dev.index)
            rows, cols = x.shape
            pairs = np.empty((rows, 2), dtype=_np_type(_acc_dtype(method, x.dtype)))
            check(lib().tf_host_reduce_rows(_lib.host_engine(dev.index), mid, _dtype_code(x.dtype), x.data_ptr(),
                                            _ptr(y), rows, cols, x.stride(0), 0 if y is None else y.stride(0),
                                            leaf_log2, pairs.ctypes.data, _stream_ptr(dev)), "tf_host_reduce_rows")
            if out is None:
                return torch.from_numpy(pairs).to(dev)
            return out.copy_(torch.from_numpy(pairs))
        if not x.is_cuda:
            x = x.to(dev, non_blocking=x.is_pinned())
        if y is not None and not y.is_cuda:
            y = y.to(dev, non_blocking=y.is_pinned())
        _lib.ensure_canary(dev.index)
        rows, cols = x.shape
        acc = _acc_dtype(method, x.dtype)
        if out is None:
            out = torch.empty(rows, 2, dtype=acc, device=dev)
        pb, cnt, _ = workspace_size(method, x.dtype, rows, cols, leaf_log2)
        parts, ctrs = _scratch.get(dev, pb, cnt)
        check(lib().tf_reduce_rows(mid, _dtype_code(x.dtype), _ptr(x), _ptr(y), rows, cols,
                                   x.stride(0), 0 if y is None else y.stride(0), leaf_log2, out.data_ptr(),
                                   _ptr(parts), pb, _ptr(ctrs), cnt, _stream_ptr(dev)), "tf_reduce_rows")
        return out


def _rows_result(method, pairs, cols) -> RowsResult:
    errors = pairs[:, 1] if method in _TWOFOLD_METHODS else torch.zeros_like(pairs[:, 1])
    return RowsResult(pairs[:, 0], errors, cols)


def sum_rows(method: Method, X, *, leaf_log2: int = 0) -> RowsResult:
    pairs = reduce_rows(method, X, leaf_log2=leaf_log2)
    return _rows_result(method, pairs, _as_rows(X).shape[1])


def dot_rows(method: Method, X, Y, *, leaf_log2: int = 0, track_product: bool = False) -> RowsResult:
    pairs = reduce_rows(method, X, Y, leaf_log2=leaf_log2, track_product=track_product)
    return _rows_result(method, pairs, _as_rows(X).shape[1])


# ---------------------------------------------------------------------------
# Error-free transforms (eft.py:28-66), evaluated by the device EFT code.

def _eft(kind: int, a, b):
    scalar_py = isinstance(a, float) and isinstance(b, float)
    tens = isinstance(a, torch.Tensor) or isinstance(b, torch.Tensor)
    if tens:
        ta = a if isinstance(a, torch.Tensor) else torch.as_tensor(a)
        tb = b if isinstance(b, torch.Tensor) else torch.as_tensor(b)
        dt = torch.promote_types(ta.dtype, tb.dtype)
    else:
        na, nb = np.asarray(a), np.asarray(b)
        ndt = np.result_type(na, nb)
        if ndt not in (np.float32, np.float64):
            ndt = np.dtype(np.float64)
        dt = torch.float32 if ndt == np.float32 else torch.float64
        ta, tb = torch.from_numpy(np.array(na, ndt)), torch.from_numpy(np.array(nb, ndt))  # keeps 0-d
    if dt not in _TORCH_OK:
        raise TypeError(f"unsupported dtype {dt}")
    ta, tb = torch.broadcast_tensors(ta.to(dt), tb.to(dt))
    dev = _device_for(ta)
    with torch.cuda.device(dev):
        _lib.ensure_canary(dev.index)
        ad = ta.to(dev).contiguous()
        bd = tb.to(dev).contiguous()
        xo = torch.empty_like(ad)
        yo = torch.empty_like(ad)
        check(lib().tf_eft(kind, _dtype_code(dt), ad.data_ptr(), bd.data_ptr(), ad.numel(), xo.data_ptr(),
                           yo.data_ptr(), _stream_ptr(dev)), "tf_eft")
    if tens:
        return Twofold(xo, yo)
    xs, ys = xo.cpu().numpy(), yo.cpu().numpy()
    if xs.ndim == 0:
        if scalar_py:
            return Twofold(float(xs), float(ys))
        t = _np_type(dt)
        return Twofold(t(xs), t(ys))
    return Twofold(xs, ys)


def fast_two_sum(a, b) -> Twofold:
    """Dekker's 3-operation EFT (eft.py:28-42).  Requires |a| >= |b| (or a == 0);
    asserted for finite scalars in debug runs, like the reference."""
    if __debug__ and np.ndim(a) == 0 and np.ndim(b) == 0 and not isinstance(a, torch.Tensor):
        fa, fb = float(a), float(b)
        if np.isfinite(fa) and np.isfinite(fb):
            assert abs(fa) >= abs(fb) or fa == 0, "fast_two_sum needs |a| >= |b|"
    return _eft(0, a, b)


def two_sum(a, b) -> Twofold:
    """Knuth's 6-operation EFT (eft.py:45-56); no ordering required."""
    return _eft(1, a, b)


def rounding_canary() -> bool:
    """True iff the device kernels evaluate EFTs under strict rounding (eft.py:59-66)."""
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device available for the device canary")
    return lib().tf_canary() == _lib.TF_OK
