"""TEST INFRASTRUCTURE — CPU oracle for the twofold hot path.

Thin ctypes wrapper over oracle/twofold_oracle.c (a C restatement of the
reference package /root/reference/pkg/src/twofold, see that file's header)
plus exact-rational tolerance checks.  Only tests/, __graft_entry__.smoke()
and bench.py's CPU-baseline legs may import this module; the product package
(paper_1401_0248_b200) never does.

Pinned by tests/test_oracle_golden.py against fixtures produced by the
reference itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from fractions import Fraction

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libtfo.so")

METHODS = ("direct", "wide", "twofold-fast", "twofold-rigorous", "kahan")
M_DIRECT, M_WIDE, M_FAST, M_RIGOROUS, M_KAHAN = range(5)
M_FAST_TP, M_RIGOROUS_TP = 5, 6  # opt-in TwoProduct dots (tf_* method | TF_TRACK_PRODUCT)
EPS = {np.dtype(np.float32): 2.0 ** -24, np.dtype(np.float64): 2.0 ** -53}

_lib = None


def build() -> str:
    """Compile the oracle library (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, i32, dp = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(ctypes.c_double)
        u64 = ctypes.c_uint64
        L.tfo_seq.argtypes = [i32, i32, vp, vp, i64, dp]
        L.tfo_lanes.argtypes = [i32, i32, vp, vp, i64, i32, dp]
        L.tfo_exact.argtypes = [i32, vp, vp, i64, i32, dp, i32]
        L.tfo_exact_f64.argtypes = [vp, i64, dp, i32]
        L.tfo_emulate_rows.argtypes = [i32, i32, vp, vp, i64, i64, i64, i64, i32, dp]
        L.tfo_emulate_leaves.argtypes = [i32, i32, vp, vp, i64, i32, dp]
        L.tfo_tree.argtypes = [i32, i32, dp, i64, dp]
        L.tfo_threads.argtypes = [i32, i32, vp, vp, i64, i32, dp]
        L.tfo_lcg_fill.argtypes = [i32, i32, u64, i32, i64, vp]
        L.tfo_leaf_log2.argtypes = [i32, i64]
        L.tfo_philox.argtypes = [ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32),
                                 ctypes.POINTER(ctypes.c_uint32)]
        L.tfo_philox.restype = None
        L.tfo_feistel.argtypes = [u64, u64, u64]
        L.tfo_feistel.restype = u64
        L.tfo_philox_fill.argtypes = [i32, i32, u64, u64, u64, i64, ctypes.c_double, ctypes.c_double,
                                      ctypes.c_double, i64, vp, i32]
        _lib = L
    return _lib


def _dt(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return 0
    if a.dtype == np.float64:
        return 1
    raise TypeError(a.dtype)


def _prep(x, y):
    x = np.ascontiguousarray(x)
    y = None if y is None else np.ascontiguousarray(y)
    return x, y, (None if y is None else y.ctypes.data)


def _acc_type(method: int, dtype):  # noqa: D103
    return np.float64 if method == M_WIDE else np.dtype(dtype).type


def _pair(method, dtype, out):
    t = _acc_type(method, dtype)
    return t(out[0]), t(out[1])


def seq(method: int, x, y=None):
    """Reference `seq` flavor (kernels.py:127-243); kahan error slot = c."""
    x, y, yp = _prep(x, y)
    out = (ctypes.c_double * 2)()
    rc = lib().tfo_seq(method, _dt(x), x.ctypes.data, yp, x.shape[0], out)
    assert rc == 0, rc
    return _pair(method, x.dtype, out)


def lanes(method: int, x, y=None, k: int = 4):
    """Reference `unroll:k` flavor (kernels.py:257-541)."""
    x, y, yp = _prep(x, y)
    out = (ctypes.c_double * 2)()
    rc = lib().tfo_lanes(method, _dt(x), x.ctypes.data, yp, x.shape[0], k, out)
    assert rc == 0, rc
    return _pair(method, x.dtype, out)


def emulate(method: int, x, y=None, leaf_log2: int = 0):
    """The GPU grid flavor's reduction tree, bit-for-bit (reduce.cu)."""
    x, y, yp = _prep(x, y)
    out = (ctypes.c_double * 2)()
    n = x.shape[0]
    rc = lib().tfo_emulate_rows(method, _dt(x), x.ctypes.data, yp, 1, n, n, n, leaf_log2, out)
    assert rc == 0, rc
    return _pair(method, x.dtype, out)


def emulate_rows(method: int, X, Y=None, leaf_log2: int = 0):
    X = np.ascontiguousarray(X)
    Y = None if Y is None else np.ascontiguousarray(Y)
    rows, cols = X.shape
    out = np.zeros(2 * rows, np.float64)
    rc = lib().tfo_emulate_rows(method, _dt(X), X.ctypes.data, None if Y is None else Y.ctypes.data,
                                rows, cols, cols, cols, leaf_log2,
                                out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert rc == 0, rc
    t = _acc_type(method, X.dtype)
    return out[0::2].astype(t), out[1::2].astype(t)


def emulate_leaves(method: int, x, y=None, leaf_log2: int = 0):
    x, y, yp = _prep(x, y)
    n = x.shape[0]
    lg = leaf_log2 or leaf_log2_auto(x.dtype, n)
    P = -(-n // (1 << lg))
    out = np.zeros(2 * max(P, 1), np.float64)
    rc = lib().tfo_emulate_leaves(method, _dt(x), x.ctypes.data, yp, n, lg,
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    assert rc == 0, rc
    t = _acc_type(method, x.dtype)
    return out[0:2 * P:2].astype(t), out[1:2 * P:2].astype(t)


def tree(method: int, dtype, pairs_s, pairs_e):
    """Balanced (padded) pair tree, as tf_merge_tree."""
    s = np.asarray(pairs_s, np.float64)
    e = np.asarray(pairs_e, np.float64)
    flat = np.empty(2 * len(s), np.float64)
    flat[0::2] = s
    flat[1::2] = e
    out = (ctypes.c_double * 2)()
    dt = 0 if np.dtype(dtype) == np.float32 else 1
    lib().tfo_tree(method, dt, flat.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(s), out)
    return _pair(method, dtype, out)


def threads(method: int, x, y=None, nthreads: int = 1):
    """Multi-thread CPU baseline: contiguous shards x reference seq + lane merge."""
    x, y, yp = _prep(x, y)
    out = (ctypes.c_double * 2)()
    lib().tfo_threads(method, _dt(x), x.ctypes.data, yp, x.shape[0], nthreads, out)
    return _pair(method, x.dtype, out)


def leaf_log2_auto(dtype, n: int) -> int:
    return lib().tfo_leaf_log2(0 if np.dtype(dtype) == np.float32 else 1, n)


def exact_components(x, y=None, absolute: bool = False, cap: int = 128, true_products: bool = False) -> tuple:
    """Exact expansion (expansion.py:79-101) of the identical addends y_i
    (true_products: of the exact products a_i*b_i, the TwoProduct target)."""
    x, y, yp = _prep(x, y)
    comp = np.zeros(cap, np.float64)
    mode = (1 if absolute else 0) | (2 if true_products else 0)
    m = lib().tfo_exact(_dt(x), x.ctypes.data, yp, x.shape[0], mode,
                        comp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap)
    assert m >= 0, "expansion overflow"
    return tuple(float(c) for c in comp[:m])


def exact_f64_components(v, cap: int = 128) -> tuple:
    v = np.ascontiguousarray(v, np.float64)
    comp = np.zeros(cap, np.float64)
    m = lib().tfo_exact_f64(v.ctypes.data, v.shape[0], comp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), cap)
    assert m >= 0
    return tuple(float(c) for c in comp[:m])


def exact(x, y=None) -> Fraction:
    return sum((Fraction(c) for c in exact_components(x, y)), Fraction(0))


def abs_sum(x, y=None) -> Fraction:
    return sum((Fraction(c) for c in exact_components(x, y, absolute=True)), Fraction(0))


def exact_true_dot(x, y) -> Fraction:
    """Exact sum of the exact products (what a TwoProduct dot tracks)."""
    return sum((Fraction(c) for c in exact_components(x, y, true_products=True)), Fraction(0))


def abs_true_dot(x, y) -> Fraction:
    return sum((Fraction(c) for c in exact_components(x, y, absolute=True, true_products=True)), Fraction(0))


def lcg_fill(kind: str, n: int, seed: int = 1, dtype=np.float64, sym: bool = False) -> np.ndarray:
    """lcg.fill restated (lcg.py:108-116); kind 'nr' or 'mmix'."""
    out = np.empty(n, dtype)
    lib().tfo_lcg_fill(0 if kind == "nr" else 1, _dt(out), seed, 1 if sym else 0, n, out.ctypes.data)
    return out


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().tfo_philox(c, k, o)
    return tuple(o)


def philox_fill(dist: str, n: int, seed: int, stream: int = 0, offset: int = 0, dtype=np.float64,
                p=(1e8, 9e8, 1e-3), total: int = 0, nthreads: int = 1) -> np.ndarray:
    """Host twin of tf_fill for the integer-exact distributions."""
    d = {"uniform01": 0, "uniform_sym": 1, "illcond": 3}[dist]
    out = np.empty(n, dtype)
    rc = lib().tfo_philox_fill(d, _dt(out), seed, stream, offset, n, p[0], p[1], p[2], total,
                               out.ctypes.data, nthreads)
    assert rc == 0
    return out


def feistel(p: int, total: int, seed: int) -> int:
    return int(lib().tfo_feistel(p, total, seed))


# ---------------------------------------------------------------------------
# Tolerances, evaluated exactly in rationals.

def deviation(v, e, S: Fraction) -> Fraction:
    """|v + e - S|: how far the twofold pair is from the exact sum."""
    return abs(Fraction(float(v)) + Fraction(float(e)) - S)


def calibrated_fast_bound(dtype, n: int, A: Fraction) -> Fraction:
    """2 N eps^2 A + 2^-6 eps A: SURVEY.md §8(c)'s calibrated twofold-fast tolerance
    for random BASELINE-size data (not a theorem; checked at N >= 2^16)."""
    eps = Fraction(EPS[np.dtype(dtype)])
    return 2 * n * eps * eps * A + Fraction(1, 64) * eps * A


def bound(method: int, dtype, n: int, A: Fraction, chain: int | None = None) -> Fraction:
    """Accuracy bound for the GPU flavor of `method` on n addends with A = sum|y|."""
    eps = Fraction(EPS[np.dtype(dtype)])
    if method == M_RIGOROUS:
        return 2 * n * eps * eps * A
    if method == M_FAST:
        # Dekker's precondition |s| >= |y| can fail on signed data;
        # each failure can lose at most about its own round-off (<= eps |y_i|),
        # hence the loose first-order term.  calibrated_fast_bound() is the tight
        # empirical one used at BASELINE sizes.
        return 2 * n * eps * eps * A + eps * A
    if method == M_KAHAN:
        return (2 * eps + 2 * n * eps * eps) * A
    # direct / wide: gamma_h with h = per-thread chain + tree depth
    if method == M_WIDE:
        eps = Fraction(2.0 ** -53)
    h = chain if chain is not None else n
    return (h * eps) / (1 - h * eps) * A
