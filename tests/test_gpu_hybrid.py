"""The hybrid host path of tf_host_reduce (csrc/host.cu hybrid_reduce + csrc/hostleaf.cpp):
host workers reduce full leaves from the back while the GPU pipeline takes chunks from
the front; the result must equal tf_reduce on the device copy bit for bit, for every
method / precision / sum-dot, pinned and pageable operands, a partial last leaf, and
whatever split the two sides' speeds produce (several reruns)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _hex(p):
    return (float(p[0]).hex(), float(p[1]).hex())


def test_hybrid_equals_device_reduce(cuda, oracle):
    import paper_1401_0248_b200 as tfb
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    eng = _lib.host_engine(0, chunk_bytes=1 << 20, threads=2)
    _lib.check(L.tf_host_engine_hybrid(eng, 4, 1 << 20), "tf_host_engine_hybrid")
    host_seen = 0
    try:
        for dt, code in ((np.float32, 0), (np.float64, 1)):
            tdt = torch.float32 if dt == np.float32 else torch.float64
            for n in ((1 << 20) + 123, 1 << 21):
                xh = oracle.lcg_fill("mmix", n, 31, dt, True)
                yh = oracle.lcg_fill("nr", n, 32, dt, True)
                xd, yd = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
                for m in ((0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)):
                    meth = list(tfb.Method)[m]
                    for dot in (False, True):
                        want = tfb.reduce(meth, xd, yd if dot else None).cpu().numpy()
                        for pinned in (False, True):
                            xs = torch.from_numpy(xh)
                            ys = torch.from_numpy(yh)
                            if pinned:
                                xs, ys = xs.pin_memory(), ys.pin_memory()
                            for _ in range(2):
                                out = np.empty(2, np.float64 if (m == 1 or dt == np.float64) else dt)
                                rc = L.tf_host_reduce(eng, m, code, xs.data_ptr(), ys.data_ptr() if dot else None, n, 0,
                                                      out.ctypes.data, None)
                                _lib.check(rc, "tf_host_reduce")
                                assert _hex(out) == _hex(want), (dt, n, m, dot, pinned)
                                gpu, host = _lib.host_split(eng)
                                assert gpu + host == n and host % 1024 == 0
                                host_seen += host
                # TwoProduct dots stay on the device path (no host leaves) and still agree
                want = tfb.reduce(tfb.Method.TWOFOLD_RIGOROUS, xd, yd, track_product=True).cpu().numpy()
                out = np.empty(2, dt)
                _lib.check(L.tf_host_reduce(eng, 3 | 0x100, code, xh.ctypes.data, yh.ctypes.data, n, 0,
                                            out.ctypes.data, None), "tf_host_reduce TP")
                assert _hex(out) == _hex(want) and _lib.host_split(eng)[1] == 0
    finally:
        L.tf_host_engine_hybrid(eng, 0, 1 << 62)
    assert host_seen > 0, "the host workers never took a leaf"


def test_hybrid_public_api_large_input(cuda, oracle):
    """Through the public API (default engine, hybrid above 8 MiB per operand): a 2^24
    binary64 numpy dot is the grid result bit for bit, and the host shared the work."""
    import paper_1401_0248_b200 as tfb
    from paper_1401_0248_b200 import _lib
    n = 1 << 24
    xh = oracle.philox_fill("uniform_sym", n, 4, 0, 0, np.float64, nthreads=8)
    yh = oracle.philox_fill("uniform_sym", n, 4, 1, 0, np.float64, nthreads=8)
    want = tfb.reduce(tfb.Method.TWOFOLD_FAST, torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda))
    r = tfb.dot_twofold_fast(xh, yh, flavor="cuda")
    assert (float(r.value).hex(), float(r.error).hex()) == _hex(want.cpu().numpy())
    gpu, host = _lib.host_split(_lib.host_engine(torch.cuda.current_device()))
    assert gpu + host == n and host > 0, (gpu, host)
    assert (float(r.value).hex(), float(r.error).hex()) == _hex(oracle.emulate(2, xh, yh))


def test_hybrid_rows_equal_device_rows(cuda, oracle):
    """tf_host_reduce_rows' hybrid path (GPU row blocks from the front, host workers whole
    rows from the back): every row pair == tf_reduce_rows on the device copy, one-leaf,
    partial-leaf and multi-leaf rows, strided pitches, pinned and pageable."""
    import paper_1401_0248_b200 as tfb
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    eng = _lib.host_engine(0, chunk_bytes=1 << 20, threads=2)
    _lib.check(L.tf_host_engine_hybrid(eng, 4, 1 << 20), "tf_host_engine_hybrid")
    host_seen = 0
    try:
        for dt, code in ((np.float32, 0), (np.float64, 1)):
            for rows, cols, ld in ((512, 4096, 4096), (300, 5000, 5003), (24, 70_001, 70_001)):
                X = oracle.lcg_fill("mmix", rows * ld, 41, dt, True).reshape(rows, ld)
                Y = oracle.lcg_fill("nr", rows * ld, 42, dt, True).reshape(rows, ld)
                Xd = torch.from_numpy(X).to(cuda)[:, :cols]
                Yd = torch.from_numpy(Y).to(cuda)[:, :cols]
                for m in ((0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)):
                    meth = list(tfb.Method)[m]
                    for dot in (False, True):
                        want = tfb.reduce_rows(meth, Xd, Yd if dot else None).cpu().numpy()
                        for pinned in (False, True):
                            xt, yt = torch.from_numpy(X), torch.from_numpy(Y)
                            if pinned:
                                xt, yt = xt.pin_memory(), yt.pin_memory()
                            out = np.empty((rows, 2), np.float64 if (m == 1 or dt == np.float64) else dt)
                            rc = L.tf_host_reduce_rows(eng, m, code, xt.data_ptr(), yt.data_ptr() if dot else None,
                                                       rows, cols, ld, ld, 0, out.ctypes.data, None)
                            _lib.check(rc, "tf_host_reduce_rows")
                            assert out.tobytes() == want.tobytes(), (dt, rows, cols, m, dot, pinned)
                            gpu, host = _lib.host_split(eng)
                            assert gpu + host == rows * cols and host % cols == 0
                            host_seen += host
    finally:
        L.tf_host_engine_hybrid(eng, 0, 1 << 62)
    assert host_seen > 0


def test_hybrid_fuzz_vs_emulator(cuda, oracle):
    """Randomised hybrid calls (sizes, misaligned host views, pinned / pageable, methods,
    precisions, sums / dots, explicit leaf sizes, 1..8 host workers) == the emulator."""
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    eng = _lib.host_engine(0, chunk_bytes=1 << 20, threads=2)
    rng = np.random.default_rng(20261021)
    try:
        for case in range(60):
            dt = np.float32 if rng.random() < 0.5 else np.float64
            code = 0 if dt == np.float32 else 1
            m = int(rng.choice((0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)))
            dot = bool(rng.random() < 0.6)
            n = int(rng.integers(1 << 13, 1 << 21))
            off = int(rng.integers(0, 4))
            lo_lg = 10 if dt == np.float32 else 9
            lg = int(rng.choice([0, 0, rng.integers(lo_lg, 15)]))
            workers = int(rng.integers(1, 9))
            _lib.check(L.tf_host_engine_hybrid(eng, workers, 1), "tf_host_engine_hybrid")
            base_x = (rng.standard_normal(n + off) * 2.0 ** rng.integers(-20, 20, n + off)).astype(dt)
            base_y = rng.uniform(-1, 1, n + off).astype(dt)
            xt, yt = torch.from_numpy(base_x), torch.from_numpy(base_y)
            if rng.random() < 0.5:
                xt, yt = xt.pin_memory(), yt.pin_memory()
            xs, ys = xt[off:], yt[off:]
            out = np.empty(2, np.float64 if (m == 1 or dt == np.float64) else dt)
            rc = L.tf_host_reduce(eng, m, code, xs.data_ptr(), ys.data_ptr() if dot else None, n, lg,
                                  out.ctypes.data, None)
            _lib.check(rc, "tf_host_reduce")
            want = oracle.emulate(m, base_x[off:], base_y[off:] if dot else None, lg)
            assert _hex(out) == _hex(want), (case, dt, m, dot, n, off, lg, workers)
    finally:
        L.tf_host_engine_hybrid(eng, 0, 1 << 62)


def test_hybrid_non_finite_matches_device(cuda, oracle):
    """inf / -inf / NaN / overflowing entries on either side of the host / GPU split: the
    hybrid pair == the device-resident pair (NaN matches NaN: payloads are not portable)."""
    import math

    import paper_1401_0248_b200 as tfb
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    eng = _lib.host_engine(0, chunk_bytes=1 << 20, threads=2)
    _lib.check(L.tf_host_engine_hybrid(eng, 4, 1), "tf_host_engine_hybrid")
    rng = np.random.default_rng(5)
    try:
        for dt, code in ((np.float32, 0), (np.float64, 1)):
            n = 1 << 20
            for pattern in ("inf_head", "inf_tail", "both", "nan", "ovf"):
                x = rng.uniform(-1, 1, n).astype(dt)
                y = rng.uniform(-1, 1, n).astype(dt)
                big = np.finfo(dt).max
                if pattern == "inf_head":
                    x[17] = np.inf
                elif pattern == "inf_tail":
                    x[n - 100] = -np.inf
                elif pattern == "both":
                    x[3], x[n - 3] = np.inf, -np.inf
                elif pattern == "nan":
                    x[n // 2] = np.nan
                else:
                    x[n - 50:n - 47] = big
                xd, yd = torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda)
                for m in ((0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)):
                    for dot in (False, True):
                        want = tfb.reduce(list(tfb.Method)[m], xd, yd if dot else None).cpu().numpy()
                        out = np.empty(2, np.float64 if (m == 1 or dt == np.float64) else dt)
                        with np.errstate(all="ignore"):
                            _lib.check(L.tf_host_reduce(eng, m, code, x.ctypes.data, y.ctypes.data if dot else None,
                                                        n, 0, out.ctypes.data, None), "tf_host_reduce")
                        for g, w in zip(out, want):
                            if math.isnan(float(w)):
                                assert math.isnan(float(g)), (dt, pattern, m, dot, out, want)
                            else:
                                assert float(g).hex() == float(w).hex(), (dt, pattern, m, dot, out, want)
                        assert _lib.host_split(eng)[1] > 0
    finally:
        L.tf_host_engine_hybrid(eng, 0, 1 << 62)
