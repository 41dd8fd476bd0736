"""Randomised parity: GPU grid flavor == the oracle's restatement of the tree, bit
for bit, over random (method, precision, sum/dot, n, leaf size, misalignment,
loader, tail, leaf split, TwoProduct); plus the reference's small-instance
criterion C6 (test_acceptance.py:180-204) on the GPU tree."""

from fractions import Fraction

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tfb(cuda):
    import paper_1401_0248_b200 as m
    torch.cuda.set_device(cuda)
    with m.using_flavor("cuda"):  # the wrappers on the grid flavor for this module
        yield m


def test_fuzz_grid_vs_emulator(tfb, oracle, cuda):
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(20261020)
    try:
        for case in range(300):
            dt = np.float32 if rng.random() < 0.5 else np.float64
            methods = (0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)
            m = int(rng.choice(methods))
            dot = bool(rng.random() < 0.6)
            tp = dot and m in (2, 3) and rng.random() < 0.3
            n = int(rng.choice([rng.integers(0, 64), rng.integers(64, 5000), rng.integers(5000, 300_000),
                                rng.integers(300_000, 2_000_000)]))
            off = int(rng.integers(0, 3))
            lo = 10 if dt == np.float32 else 9
            lg = int(rng.choice([0, 0, rng.integers(lo, 18)]))
            scale = 2.0 ** rng.integers(-30, 30)
            xh = (rng.standard_normal(n + off) * scale * 2.0 ** rng.integers(-8, 8, n + off)).astype(dt)
            yh = rng.uniform(-1, 1, n + off).astype(dt)
            x, y = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
            L.tf_set_loader(int(rng.choice([0, 1, 2, 3, 6, 7, 8])))
            L.tf_set_tail(int(rng.choice([0, 1, 2])))
            L.tf_set_leaf_split(int(rng.choice([0, 1, 2, 4])))
            meth = list(tfb.Method)[m]
            got = tfb.reduce(meth, x[off:], y[off:] if dot else None, leaf_log2=lg, track_product=tp).cpu().numpy()
            want = oracle.emulate(m + (3 if tp else 0), xh[off:], yh[off:] if dot else None, lg)
            assert float(got[0]).hex() == float(want[0]).hex() and float(got[1]).hex() == float(want[1]).hex(), \
                (case, dt, m, dot, tp, n, off, lg, got, want)
    finally:
        L.tf_set_loader(0)
        L.tf_set_tail(0)
        L.tf_set_leaf_split(0)


def test_fuzz_rows_vs_emulator(tfb, oracle, cuda):
    """Random row-wise reductions (rows x cols, leading dimension / offset, leaf size,
    method, sum/dot, TwoProduct, rows kernel auto / CTA per row / lane groups) == the
    oracle's per-row restatement of the tree, bit for bit."""
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(20261021)
    try:
        for case in range(120):
            dt = np.float32 if rng.random() < 0.5 else np.float64
            methods = (0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)
            m = int(rng.choice(methods))
            dot = bool(rng.random() < 0.6)
            tp = dot and m in (2, 3) and rng.random() < 0.3
            rows = int(rng.integers(2, 400))
            cols = int(rng.choice([rng.integers(1, 40), rng.integers(40, 1100), rng.integers(1100, 9000)]))
            pad = int(rng.choice([0, 0, rng.integers(1, 9)]))
            off = int(rng.integers(0, 2))
            lo = 10 if dt == np.float32 else 9
            lg = int(rng.choice([0, 0, rng.integers(lo, 15)]))
            ld = cols + pad
            bx = (rng.standard_normal(rows * ld + off) * 2.0 ** rng.integers(-10, 10, rows * ld + off)).astype(dt)
            by = rng.uniform(-1, 1, rows * ld + off).astype(dt)
            X = torch.from_numpy(bx).to(cuda)[off:].as_strided((rows, cols), (ld, 1))
            Y = torch.from_numpy(by).to(cuda)[off:].as_strided((rows, cols), (ld, 1))
            Xh = np.ascontiguousarray(X.cpu().numpy())
            Yh = np.ascontiguousarray(Y.cpu().numpy())
            kind = int(rng.choice([0, 1, 2]))
            L.tf_set_rows_kernel(kind)
            meth = list(tfb.Method)[m]
            got = tfb.reduce_rows(meth, X, Y if dot else None, leaf_log2=lg, track_product=tp).cpu().numpy()
            ev, ee = oracle.emulate_rows(m + (3 if tp else 0), Xh, Yh if dot else None, lg)
            for r in range(rows):
                assert float(got[r, 0]).hex() == float(ev[r]).hex() and float(got[r, 1]).hex() == float(ee[r]).hex(), \
                    (case, dt, m, dot, tp, rows, cols, ld, off, lg, kind, r, L.tf_last_launch().decode())
    finally:
        L.tf_set_rows_kernel(0)


def test_small_instance_criterion_c6_on_the_grid(tfb, oracle):
    """|v + e - S| <= 2 eps |S| for the rigorous grid flavor on the reference's C6 instances."""
    def check(data, eps):
        r = tfb.sum_twofold_rigorous(data)
        got = Fraction(float(r.value)) + Fraction(float(r.error))
        exact = sum((Fraction(float(v)) for v in data), Fraction(0))
        assert abs(got - exact) <= 2 * Fraction(eps) * abs(exact), (data, r)

    mags = [1.0, 2.0 ** -24, 3.25, 7.1e-3, 2.0 ** 20]
    for bits in range(32):
        signed = [(-m if bits >> i & 1 else m) for i, m in enumerate(mags)]
        check(np.array(signed, np.float64), 2.0 ** -53)
        check(np.array(signed, np.float32), 2.0 ** -24)
    rng = np.random.default_rng(6)
    for _ in range(300):
        n = int(rng.integers(1, 21))
        data = (rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-8, 8, n))
        check(data.astype(np.float32), 2.0 ** -24)


def test_every_loader_every_chain_length(tfb, oracle, cuda):
    """Systematic: every loader (LDG, LDG deep, four TMA ring shapes) x precision x
    sum/dot x method x leaf size from one vector per chain (R = 1) up to R = 32 —
    in particular R below the loader's batch depth U — bit-identical to the emulator."""
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(77)
    try:
        for dt in (np.float32, np.float64):
            floor = 10 if dt == np.float32 else 9
            for lg in range(floor, floor + 6):
                n = (1 << lg) * 37 + int(rng.integers(1, 1 << lg))
                xh = (rng.standard_normal(n) * 2.0 ** rng.integers(-6, 6, n)).astype(dt)
                yh = rng.uniform(-1, 1, n).astype(dt)
                x, y = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
                for m in ((0, 2, 3, 4) if dt == np.float64 else (0, 1, 2, 3, 4)):
                    meth = list(tfb.Method)[m]
                    for dot in (False, True):
                        want = oracle.emulate(m, xh, yh if dot else None, lg)
                        for loader in (1, 8, 2, 3, 6, 7):
                            L.tf_set_loader(loader)
                            got = tfb.reduce(meth, x, y if dot else None, leaf_log2=lg).cpu().numpy()
                            assert float(got[0]).hex() == float(want[0]).hex() and \
                                float(got[1]).hex() == float(want[1]).hex(), (dt, lg, m, dot, loader, got, want)
    finally:
        L.tf_set_loader(0)
