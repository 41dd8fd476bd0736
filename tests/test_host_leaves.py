"""The hybrid host path's CPU leaf reducer (csrc/hostleaf.cpp via tf_host_leaves) on CPU:
its leaf pairs must be exactly the device leaves' — the oracle's restatement of the
GPU tree (oracle.emulate_leaves) — for every method, precision, sum/dot and leaf size,
on data with wide exponent ranges, subnormals, signed zeros and cancellation."""

import ctypes

import numpy as np
import pytest

from paper_1401_0248_b200 import _lib


def _host_leaves(m, x, y, lg, lo, hi):
    L = _lib.lib()
    dt = 0 if x.dtype == np.float32 else 1
    acc = np.float64 if (m == 1 or dt == 1) else np.float32
    out = np.zeros(2 * (hi - lo), acc)
    rc = L.tf_host_leaves(m, dt, x.ctypes.data, None if y is None else y.ctypes.data, x.shape[0], lg, lo, hi,
                          out.ctypes.data)
    _lib.check(rc, "tf_host_leaves")
    return out[0::2], out[1::2]


def _data(rng, n, dt, kind):
    if kind == "wide":
        v = rng.standard_normal(n) * 2.0 ** rng.integers(-40, 40, n)
    elif kind == "subnormal":
        tiny = np.finfo(dt).tiny
        v = rng.standard_normal(n) * tiny * 2.0 ** rng.integers(-20, 4, n)
        v[::7] = -0.0
    elif kind == "cancel":
        v = rng.uniform(1e6, 1e7, n)
        v[1::2] = -v[0::2][: v[1::2].shape[0]] * (1 + 2.0 ** -20)
    else:
        v = rng.uniform(-1, 1, n)
    return v.astype(dt)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
@pytest.mark.parametrize("kind", ["uniform", "wide", "subnormal", "cancel"])
def test_host_leaves_equal_device_leaves(oracle, dt, kind):
    rng = np.random.default_rng(abs(hash((dt().itemsize, kind))) % 2**32)
    lo_lg = 10 if dt == np.float32 else 9
    for lg in (lo_lg, lo_lg + 2, 16):
        L = 1 << lg
        n = 3 * L + 17  # three full leaves and a partial one (the host takes full leaves only)
        x = _data(rng, n, dt, kind)
        y = _data(rng, n, dt, "wide")
        for m in ((0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)):
            for yy in (None, y):
                want_s, want_e = oracle.emulate_leaves(m, x, yy, lg)
                got_s, got_e = _host_leaves(m, x, yy, lg, 0, 3)
                assert got_s.tobytes() == want_s[:3].astype(got_s.dtype).tobytes(), (dt, kind, lg, m, yy is None)
                assert got_e.tobytes() == want_e[:3].astype(got_e.dtype).tobytes(), (dt, kind, lg, m, yy is None)
                s1, e1 = _host_leaves(m, x, yy, lg, 1, 3)  # a sub-range lands at its own offsets
                assert s1.tobytes() == got_s[1:].tobytes() and e1.tobytes() == got_e[1:].tobytes()


def test_host_leaves_validates():
    L = _lib.lib()
    x = np.zeros(4096, np.float64)
    out = np.zeros(64)
    assert L.tf_host_leaves(2, 1, x.ctypes.data, None, 4096, 9, 0, 9, out.ctypes.data) == _lib.TF_EINVAL_ARG  # past n
    assert L.tf_host_leaves(1, 1, x.ctypes.data, None, 4096, 9, 0, 1, out.ctypes.data) == _lib.TF_EINVAL_DTYPE  # wide f64
    assert L.tf_host_leaves(5, 1, x.ctypes.data, None, 4096, 9, 0, 1, out.ctypes.data) == _lib.TF_EINVAL_METHOD  # TP
    assert L.tf_host_leaves(2, 1, x.ctypes.data, None, 4096, 8, 0, 1, out.ctypes.data) == _lib.TF_EINVAL_ARG  # leaf < 256V
    assert L.tf_host_leaves(2, 1, x.ctypes.data, None, 4096, 9, 0, 8, ctypes.c_void_p(out.ctypes.data)) == _lib.TF_OK


def test_baseline_build_gives_the_same_bits():
    """The x86-64 baseline build of hostleaf.cpp (TFB_HOSTLEAF_BASE=1) == the AVX-512 build."""
    import os
    import subprocess
    import sys
    code = ("import numpy as np, sys; sys.path[:0] = [%r, %r]; from test_host_leaves import _host_leaves;"
            "rng = np.random.default_rng(5); x = (rng.standard_normal(4 * 4096) * 2.0 ** rng.integers(-30, 30, 4 * 4096));"
            "y = rng.uniform(-1, 1, 4 * 4096);"
            "outs = [_host_leaves(m, a.astype(t), None if b is None else b.astype(t), 12, 0, 4) for t in (np.float32, np.float64)"
            " for m in ((0, 1, 2, 3, 4) if t == np.float32 else (0, 2, 3, 4)) for a, b in ((x, None), (x, y))];"
            "print(b''.join(s.tobytes() + e.tobytes() for s, e in outs).hex())")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    runs = [subprocess.run([sys.executable, "-c", code % (repo, os.path.join(repo, "tests"))], env=dict(os.environ, **extra), capture_output=True,
                           text=True, check=True, cwd=repo).stdout for extra in ({}, {"TFB_HOSTLEAF_BASE": "1"})]
    assert runs[0] == runs[1] and len(runs[0]) > 1000


def _host_rows(m, X, Y, lg, lo, hi, cols, ld):
    L = _lib.lib()
    dt = 0 if X.dtype == np.float32 else 1
    acc = np.float64 if (m == 1 or dt == 1) else np.float32
    out = np.zeros(2 * (hi - lo), acc)
    rows = X.shape[0] if X.ndim == 2 else 1
    rc = L.tf_host_rows(m, dt, X.ctypes.data, None if Y is None else Y.ctypes.data, rows, cols, ld, ld, lg, lo, hi,
                        out.ctypes.data)
    _lib.check(rc, "tf_host_rows")
    return out[0::2], out[1::2]


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_host_rows_equal_device_rows(oracle, dt):
    """The hybrid rows path's CPU row reducer == the emulator's per-row tree: one-leaf rows
    (full and partial leaves), multi-leaf rows (leaf tree padded to a power of two, a
    partial last leaf), strided leading dimensions, sums and dots, every method."""
    rng = np.random.default_rng(11 if dt == np.float32 else 12)
    lo_lg = 10 if dt == np.float32 else 9
    for rows, cols, pad, lg in ((7, 1 << lo_lg, 0, lo_lg), (5, 777, 3, lo_lg), (4, 3 * (1 << lo_lg) + 5, 1, lo_lg),
                                (6, 100, 0, lo_lg + 2), (3, 5 * (1 << lo_lg), 0, lo_lg), (2, 1, 0, lo_lg)):
        ld = cols + pad
        Xb = _data(rng, rows * ld, dt, "wide").reshape(rows, ld)
        Yb = _data(rng, rows * ld, dt, "uniform").reshape(rows, ld)
        Xc, Yc = np.ascontiguousarray(Xb[:, :cols]), np.ascontiguousarray(Yb[:, :cols])
        for m in ((0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)):
            for yy, yyc in ((None, None), (Yb, Yc)):
                ev, ee = oracle.emulate_rows(m, Xc, yyc, lg)
                gs, ge = _host_rows(m, Xb, yy, lg, 0, rows, cols, ld)
                assert gs.tobytes() == ev.astype(gs.dtype).tobytes(), (dt, rows, cols, pad, lg, m, yy is None)
                assert ge.tobytes() == ee.astype(ge.dtype).tobytes(), (dt, rows, cols, pad, lg, m, yy is None)
                s1, e1 = _host_rows(m, Xb, yy, lg, 1, rows, cols, ld)  # a sub-range of rows
                assert s1.tobytes() == gs[1:].tobytes() and e1.tobytes() == ge[1:].tobytes()
