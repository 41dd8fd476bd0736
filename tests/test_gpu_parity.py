"""GPU parity: the CUDA path through the C ABI vs the oracle (run on a B200).

* grid ("cuda") flavor == the oracle's restatement of the GPU tree, bit for bit,
  for every method x precision x {sum, dot}, ragged / empty / misaligned inputs
  and explicit leaf sizes; plus the exact-sum tolerances of SURVEY.md §8(c)
* seq and unroll:k flavors == the REFERENCE's own outputs (golden fixtures)
* reruns bit-identical; rows == per-row 1-D; streamed host path == device path
* Philox device fills == host twin; shard trees == single-GPU tree
"""

import numpy as np
import pytest
import torch

from golden_inputs import load_inputs

pytestmark = pytest.mark.gpu

METHOD_ID = {"direct": 0, "wide": 1, "twofold-fast": 2, "twofold-rigorous": 3, "kahan": 4}
SIZES = [0, 1, 2, 3, 5, 17, 255, 256, 1023, 1024, 1025, 4095, 4096, 4097, 8191, 8192, 8193,
         65536 + 3, (1 << 18) + 1, (1 << 20) + 7]


@pytest.fixture(scope="module")
def tfb(cuda):
    """The package with the wrappers switched to the grid flavor for this module
    (their default is the reference's seq bits; tests/test_gpu_dropin.py covers that)."""
    import paper_1401_0248_b200 as m
    torch.cuda.set_device(cuda)
    with m.using_flavor("cuda"):
        yield m


def _methods(dt):
    return (0, 1, 2, 3, 4) if dt == np.float32 else (0, 2, 3, 4)


def _hex(v):
    return float(v).hex()


def _same(got, want, ctx):
    assert _hex(got[0]) == _hex(want[0]) and _hex(got[1]) == _hex(want[1]), (ctx, got, want)


def test_canary(tfb):
    assert tfb.rounding_canary()


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_grid_matches_emulator_all_methods(tfb, oracle, cuda, dt):
    for n in SIZES:
        xh = oracle.lcg_fill("mmix", n, 3 + n % 7, dt, True)
        yh = oracle.lcg_fill("nr", n, 5 + n % 5, dt, True)
        x, y = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
        for m in _methods(dt):
            meth = list(tfb.Method)[m]
            _same(tfb.reduce(meth, x).cpu().numpy(), oracle.emulate(m, xh), (m, dt, n, "sum"))
            _same(tfb.reduce(meth, x, y).cpu().numpy(), oracle.emulate(m, xh, yh), (m, dt, n, "dot"))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_explicit_leaf_sizes_and_misaligned_views(tfb, oracle, cuda, dt):
    n = 100_003
    xh = oracle.lcg_fill("mmix", n + 1, 9, dt, True)
    yh = oracle.lcg_fill("nr", n + 1, 10, dt, False)
    xb, yb = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
    lo = 10 if dt == np.float32 else 9
    for lg in (lo, lo + 2, 14, 16, 20):
        for m in _methods(dt):
            meth = list(tfb.Method)[m]
            # aligned
            _same(tfb.reduce(meth, xb[:n], yb[:n], leaf_log2=lg).cpu().numpy(),
                  oracle.emulate(m, xh[:n], yh[:n], lg), (m, lg, "aligned"))
            # 1-element offset: not 16-byte aligned -> scalar-load kernel, same tree
            _same(tfb.reduce(meth, xb[1:], yb[1:], leaf_log2=lg).cpu().numpy(),
                  oracle.emulate(m, xh[1:], yh[1:], lg), (m, lg, "misaligned"))


def test_reruns_bit_identical(tfb, cuda):
    x = tfb.philox_fill("normal", 1 << 24, seed=1, stream=0, dtype=torch.float32)
    y = tfb.philox_fill("normal", 1 << 24, seed=1, stream=1, dtype=torch.float32)
    for meth in tfb.Method:
        first = tfb.reduce(meth, x, y).cpu()
        for _ in range(10):
            assert torch.equal(tfb.reduce(meth, x, y).cpu(), first), meth


def test_value_channel_shared_by_direct_fast_rigorous(tfb, oracle, cuda):
    # GPU analogue of test_kernels.py:129-135 / test_acceptance.py:119-130
    for dt in (np.float32, np.float64):
        for seed in range(1, 11):
            xh = oracle.lcg_fill("mmix", 50_000, seed, dt, True)
            x = torch.from_numpy(xh).to(cuda)
            d = tfb.sum_direct(x).value
            assert tfb.sum_twofold_fast(x).value.tobytes() == d.tobytes()
            assert tfb.sum_twofold_rigorous(x).value.tobytes() == d.tobytes()


def test_dot_by_ones_equals_sum_bitwise(tfb, oracle, cuda):
    # test_kernels.py:102-111 on the grid flavor
    xh = oracle.lcg_fill("nr", 123_457, 1, np.float32, False)
    x = torch.from_numpy(xh).to(cuda)
    ones = torch.ones_like(x)
    for dotf, sumf in ((tfb.dot_twofold_fast, tfb.sum_twofold_fast), (tfb.dot_twofold_rigorous,
                       tfb.sum_twofold_rigorous), (tfb.dot_kahan, tfb.sum_kahan), (tfb.dot_direct, tfb.sum_direct)):
        assert dotf(x, ones).twofold == sumf(x).twofold
    assert tfb.dot_wide(x, ones).value == tfb.sum_wide(x).value


def test_non_finite_flavors_match_reference(tfb, oracle, golden):
    """GPU seq / unroll:k / vec on inf / -inf / NaN / overflow inputs == the
    reference's run_flavor (tests/golden nonfinite section; NaN == NaN)."""
    inputs = load_inputs(oracle, golden, "nonfinite")
    for case in golden["nonfinite"]["cases"]:
        x, y = inputs[case["input"]]
        r = tfb.run_flavor(tfb.Method(case["method"]), tfb.Flavor.parse(case["flavor"]), x, y)
        assert _hex(r.value) == case["value"] and _hex(r.error) == case["error"], case


def test_seq_and_lane_flavors_bit_exact_with_reference(tfb, oracle, golden):
    """GPU seq / unroll:k / vec == the reference's own run_flavor output (fixtures)."""
    inputs = load_inputs(oracle, golden)
    checked = 0
    for case in golden["cases"]:
        if case["n"] > 20_000:
            continue  # the one-thread seq kernel is slow; large inputs are covered by the tree tests
        x, y = inputs[case["input"]]
        meth = tfb.Method(case["method"])
        r = tfb.run_flavor(meth, tfb.Flavor.parse(case["flavor"]), x, y)
        assert _hex(r.value) == case["value"] and _hex(r.error) == case["error"], case
        assert type(r.value).__name__ == case["value_type"]
        assert r.adds_performed == case["adds"]
        checked += 1
    assert checked > 1000


def test_hours100_on_gpu_seq(tfb):
    """accuracy.run_hours100's goldens (test_acceptance.py:46-60) from the GPU seq flavor."""
    data = np.full(3_600_000, np.float32(0.1), np.float32)
    seq = tfb.Flavor.sequential()
    d = float(tfb.run_flavor(tfb.Method.DIRECT, seq, data).value) / 3600
    t = tfb.run_flavor(tfb.Method.TWOFOLD_FAST, seq, data)
    th = (float(t.value) + float(t.error)) / 3600
    assert abs(d - 96.3958) <= 0.0005
    assert abs(th - 99.9359) <= 0.001
    assert abs(float(t.error) / 3600 - 3.54008) <= 0.01
    # the grid flavor on the same data: v+e is exact to the binary32 EFT level
    g = tfb.sum_twofold_fast(data)
    assert abs((float(g.value) + float(g.error)) / 3600 - 100.0) < 1e-4


def test_tolerances_against_exact_oracle(tfb, oracle, cuda):
    cases = [("uniform01", np.float64, None, 1 << 20), ("uniform_sym", np.float64, "y", 1 << 20),
             ("uniform_sym", np.float32, "y", 1 << 22), ("uniform01", np.float32, None, 1 << 22)]
    for dist, dt, dot, n in cases:
        tdt = torch.float32 if dt == np.float32 else torch.float64
        x = tfb.philox_fill(dist, n, seed=7, stream=0, dtype=tdt)
        y = tfb.philox_fill(dist, n, seed=7, stream=1, dtype=tdt) if dot else None
        xh = x.cpu().numpy()
        yh = None if y is None else y.cpu().numpy()
        S, A = oracle.exact(xh, yh), oracle.abs_sum(xh, yh)
        for m in (2, 3, 4, 0):
            pair = tfb.reduce(list(tfb.Method)[m], x, y).cpu().numpy()
            if m in (2, 3):
                dev = oracle.deviation(pair[0], pair[1], S)
            else:
                dev = oracle.deviation(pair[0], 0.0, S)
            chain = (1 << tfb.leaf_log2_for(tdt, n)) // 256 + 30
            assert dev <= oracle.bound(m, dt, n, A, chain=chain), (dist, dt, m, float(dev))
            if m == 2:  # twofold-fast: the calibrated tolerance of SURVEY.md §8(c) at these sizes
                assert dev <= oracle.calibrated_fast_bound(dt, n, A), (dist, dt, float(dev))


def test_rows_equal_per_row_reduce_and_emulator(tfb, oracle, cuda):
    for dt, rows, cols in ((np.float32, 37, 70_001), (np.float64, 5, 300_000), (np.float32, 300, 4096),
                           (np.float32, 8, 1)):
        tdt = torch.float32 if dt == np.float32 else torch.float64
        X = tfb.rows_scaled_normal(rows, cols, seed=3, stream=0, dtype=tdt)
        Y = tfb.rows_scaled_normal(rows, cols, seed=3, stream=1, dtype=tdt)
        Xh, Yh = X.cpu().numpy(), Y.cpu().numpy()
        for m in _methods(dt):
            meth = list(tfb.Method)[m]
            got = tfb.reduce_rows(meth, X, Y).cpu().numpy()
            ev, ee = oracle.emulate_rows(m, Xh, Yh)
            for r in range(rows):
                _same(got[r], (ev[r], ee[r]), (dt, rows, cols, m, r))
            lg = tfb.leaf_log2_for(tdt, rows * cols)  # the rows auto leaf depends on rows*cols
            for r in (0, rows - 1):
                _same(got[r], tfb.reduce(meth, X[r], Y[r], leaf_log2=lg).cpu().numpy(), ("row vs 1-D", r))


def test_misaligned_binary32_shifted_loads(tfb, oracle, cuda):
    """binary32 operands 1..3 elements past a 16-byte boundary (shared offset) take the
    shifted-vector loads (aligned LDG + one lane shuffle; lane 31 reads the next warp's
    elements): bit-identical to the emulator for every method x sum/dot x TwoProduct, full
    and partial leaves, explicit leaf sizes, and rows whose pitch keeps the offset."""
    L = tfb._lib.lib()
    for n in (4096 * 3 + 5, 100_003, (1 << 20) + 77):
        xh = oracle.lcg_fill("mmix", n + 8, 81, np.float32, True)
        yh = oracle.lcg_fill("nr", n + 8, 82, np.float32, True)
        xd, yd = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
        for off in (1, 2, 3):
            x, y = xd[off:off + n], yd[off:off + n]
            xs, ys = xh[off:off + n], yh[off:off + n]
            cases = [(m, list(tfb.Method)[m], False) for m in (0, 1, 2, 3, 4)]
            cases += [(5, tfb.Method.TWOFOLD_FAST, True), (6, tfb.Method.TWOFOLD_RIGOROUS, True)]
            for m, meth, tp in cases:
                for yy, yyh in ((None, None), (y, ys)):
                    if tp and yy is None:
                        continue
                    for lg in (0, 12):
                        got = tfb.reduce(meth, x, yy, leaf_log2=lg, track_product=tp).cpu().numpy()
                        if lg == 0 and n > 100_000:
                            assert f"shift{off}" in L.tf_last_launch().decode(), L.tf_last_launch().decode()
                        _same(got, oracle.emulate(m, xs, yyh, lg), (n, off, m, tp, yy is None, lg))
    # rows: pitch 4100 floats (16-byte multiple), base 2 elements in -> every row shifted by 2
    base = torch.from_numpy(oracle.lcg_fill("mmix", 40 * 4100 + 8, 83, np.float32, True)).to(cuda)
    X = base[2:2 + 40 * 4100].view(40, 4100)[:, :4099]
    Xh = np.ascontiguousarray(X.cpu().numpy())
    for m in (2, 3, 4):
        L.tf_set_rows_kernel(1)
        try:
            got = tfb.reduce_rows(list(tfb.Method)[m], X, leaf_log2=10).cpu().numpy()
            assert "shift2" in L.tf_last_launch().decode(), L.tf_last_launch().decode()
        finally:
            L.tf_set_rows_kernel(0)
        ev, ee = oracle.emulate_rows(m, Xh, None, 10)
        for r in range(40):
            _same(got[r], (ev[r], ee[r]), ("rows", m, r))


SHORT_COLS = [1, 3, 4, 7, 16, 31, 33, 64, 100, 128, 255, 256, 257, 1000, 1024, 1025, 2049, 4095, 4096]


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_rows_short_kernel_matches_emulator(tfb, oracle, cuda, dt):
    """rows.cuh (lane groups of 1..32 per row, every row inside one leaf) == the oracle's
    restatement of the 256-chain leaf tree, bit for bit, for every method x sum/dot x
    TwoProduct; == the CTA-per-leaf kernel incl. signed zeros (all -0 rows, zero rows);
    aligned, strided-aligned and misaligned (scalar path) leading dimensions.  Leaf 2^13, so
    every row fits one leaf and the longer rows take several vectors per chain (K = 2..8)."""
    L = tfb._lib.lib()
    tdt = torch.float32 if dt == np.float32 else torch.float64
    try:
        for cols in SHORT_COLS:
            rows = 67
            Xh = oracle.lcg_fill("mmix", rows * cols, 40 + cols % 11, dt, True).reshape(rows, cols)
            Yh = oracle.lcg_fill("nr", rows * cols, 50 + cols % 7, dt, True).reshape(rows, cols)
            Xh[5] = -0.0  # a row summing to -0 in every order
            Xh[6] = 0.0
            Xh[7, 1::2] = -Xh[7, 0::2][: Xh[7, 1::2].shape[0]]  # cancelling neighbours
            X, Y = torch.from_numpy(Xh).to(cuda), torch.from_numpy(Yh).to(cuda)
            cases = [(m, list(tfb.Method)[m], False) for m in _methods(dt)]
            cases += [(5, tfb.Method.TWOFOLD_FAST, True), (6, tfb.Method.TWOFOLD_RIGOROUS, True)]
            for m, meth, tp in cases:
                for yy, yyh in ((None, None), (Y, Yh)):
                    if tp and yy is None:
                        continue
                    ev, ee = oracle.emulate_rows(m, Xh, yyh, leaf_log2=13)
                    L.tf_set_rows_kernel(2)
                    got = tfb.reduce_rows(meth, X, yy, leaf_log2=13, track_product=tp).cpu().numpy()
                    desc = L.tf_last_launch().decode()
                    assert "rows_short_kernel" in desc, (dt, cols, m, desc)
                    L.tf_set_rows_kernel(1)
                    cta = tfb.reduce_rows(meth, X, yy, leaf_log2=13, track_product=tp).cpu().numpy()
                    assert np.array_equal(got.view(np.uint8), cta.view(np.uint8)), (dt, cols, m, yy is None)
                    for r in range(rows):
                        _same(got[r], (ev[r], ee[r]), (dt, cols, m, r, yy is None))
        # leading dimensions: aligned ld > cols (vector path) and a 1-element offset (scalar path)
        base = torch.from_numpy(oracle.lcg_fill("mmix", 41 * 1040, 61, dt, True).reshape(41, 1040)).to(cuda)
        for view in (base[:, :1000], base[:, 1:1001], base[:, 3:20]):
            vh = np.ascontiguousarray(view.cpu().numpy())
            for m in (2, 3, 4):
                L.tf_set_rows_kernel(2)
                got = tfb.reduce_rows(list(tfb.Method)[m], view).cpu().numpy()
                ev, ee = oracle.emulate_rows(m, vh)
                for r in range(41):
                    _same(got[r], (ev[r], ee[r]), (dt, view.shape, view.storage_offset(), m, r))
    finally:
        L.tf_set_rows_kernel(0)
    # the auto choice takes the lane-group kernel for short rows
    tfb.reduce_rows(tfb.Method.TWOFOLD_FAST, torch.ones(1000, 64, dtype=tdt, device=cuda))
    assert "rows_short_kernel" in L.tf_last_launch().decode()


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_sequential_flavors_streamed_match_reference_order(tfb, oracle, cuda, dt):
    """seq and unroll:k on inputs large enough for the bulk-copy ring (seqpipe.cuh):
    bit-identical to the oracle's restatement of the reference kernels, for every
    method x sum/dot x TwoProduct, head misalignment 0..3 elements (operands with equal
    and with different offsets mod 16 bytes, the latter on the plain kernels)."""
    for n, offx, offy in ((40_000, 0, 0), (100_003, 1, 1), (70_001, 3, 3), (50_000, 1, 2), (1 << 18, 2, 2)):
        xh = oracle.lcg_fill("mmix", n + 4, 71 + offx, dt, True)
        yh = oracle.lcg_fill("nr", n + 4, 72 + offy, dt, True)
        xd, yd = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
        x, y = xd[offx:offx + n], yd[offy:offy + n]
        xs, ys = xh[offx:offx + n], yh[offy:offy + n]
        cases = [(m, list(tfb.Method)[m], False) for m in _methods(dt)]
        cases += [(5, tfb.Method.TWOFOLD_FAST, True), (6, tfb.Method.TWOFOLD_RIGOROUS, True)]
        for m, meth, tp in cases:
            for yy, yyh in ((None, None), (y, ys)):
                if tp and yy is None:
                    continue
                got = tfb.reduce(meth, x, yy, flavor=tfb.Flavor.sequential(), track_product=tp).cpu().numpy()
                _same(got, oracle.seq(m, xs, yyh), (dt, n, offx, offy, m, "seq"))
                for k in (2, 4, 16):
                    got = tfb.reduce(meth, x, yy, flavor=tfb.Flavor.unrolled(k), track_product=tp).cpu().numpy()
                    _same(got, oracle.lanes(m, xs, yyh, k), (dt, n, offx, offy, m, "lanes", k))


def test_sharded_rows_single_rank_is_reduce_rows(tfb, oracle, cuda):
    """dist.sharded_rows at world size 1 (no process group): the device kernels with the whole
    matrix's leaf size, == reduce_rows == the emulator."""
    rows, cols = 41, 7000
    Xh = oracle.lcg_fill("mmix", rows * cols, 91, np.float32, True).reshape(rows, cols)
    Yh = oracle.lcg_fill("nr", rows * cols, 92, np.float32, True).reshape(rows, cols)
    X, Y = torch.from_numpy(Xh).to(cuda), torch.from_numpy(Yh).to(cuda)
    got = tfb.sharded_rows(tfb.Method.TWOFOLD_RIGOROUS, X, Y, rows_global=rows, gather=True).cpu().numpy()
    ref = tfb.reduce_rows(tfb.Method.TWOFOLD_RIGOROUS, X, Y).cpu().numpy()
    assert np.array_equal(got.view(np.uint8), ref.view(np.uint8))
    ev, ee = oracle.emulate_rows(3, Xh, Yh)
    for r in range(rows):
        _same(got[r], (ev[r], ee[r]), r)
    with pytest.raises(ValueError):
        tfb.sharded_rows(tfb.Method.DIRECT, X[:5], rows_global=rows)


def test_rows_strided_leading_dimension(tfb, oracle, cuda):
    base = tfb.rows_scaled_normal(9, 5000, seed=4, stream=0, dtype=torch.float32)
    X = base[:, :4999]  # ld = 5000 > cols: 4-byte misaligned rows -> scalar path
    got = tfb.reduce_rows(tfb.Method.TWOFOLD_FAST, X).cpu().numpy()
    Xh = np.ascontiguousarray(X.cpu().numpy())
    ev, ee = oracle.emulate_rows(2, Xh)
    for r in range(9):
        _same(got[r], (ev[r], ee[r]), r)


def test_streamed_host_path_equals_device_path(tfb, oracle, cuda):
    """Host-buffer engine (tf_host_reduce): 1 MiB chunks force 17 chunks of 16
    leaves; pageable and pinned inputs, sums and dots, equal the emulator."""
    from paper_1401_0248_b200 import _lib, api
    eng = _lib.host_engine(0, chunk_bytes=1 << 20, threads=3)
    dev = torch.device("cuda", 0)
    n = (1 << 21) + 5
    xh = oracle.lcg_fill("mmix", n, 21, np.float64, True)
    yh = oracle.lcg_fill("nr", n, 22, np.float64, True)
    for pinned in (False, True):
        xt, yt = torch.from_numpy(xh), torch.from_numpy(yh)
        if pinned:
            xt, yt = xt.pin_memory(), yt.pin_memory()
        for m in (0, 2, 3, 4):
            meth = list(tfb.Method)[m]
            got = api._host_pair(meth, xt, yt, dev, engine=eng)
            _same(got, oracle.emulate(m, xh, yh), (m, pinned))
            got = api._host_pair(meth, xt, None, dev, engine=eng)
            _same(got, oracle.emulate(m, xh), (m, pinned, "sum"))
        got = api._host_pair(tfb.Method.TWOFOLD_FAST, xt[:0], None, dev, engine=eng)
        assert got.tolist() == [0.0, 0.0]
        # small inputs take the zero-copy path (kernel reads page-locked host memory):
        # whole buffers and interior slices of them
        for a, b in ((0, 4097), (3, 9000), (1000, 1000 + (1 << 15))):
            for m in (2, 3):
                meth = list(tfb.Method)[m]
                got = api._host_pair(meth, xt[a:b], yt[a:b], dev, engine=eng)
                _same(got, oracle.emulate(m, xh[a:b], yh[a:b]), (m, pinned, a, b, "zero-copy"))
    xf = xh.astype(np.float32)
    got = api._host_pair(tfb.Method.WIDE, torch.from_numpy(xf), None, dev, engine=eng)
    _same(got, oracle.emulate(1, xf), "wide")
    r = tfb.dot_twofold_fast(xh, yh)  # numpy inputs through the public wrapper (default engine)
    _same((r.value, r.error), oracle.emulate(2, xh, yh), "wrapper")
    got = tfb.reduce(tfb.Method.KAHAN, torch.from_numpy(xh)).cpu().numpy()
    _same(got, oracle.emulate(4, xh), "reduce host")
    # an explicit leaf (2^21 f64 = 16 MiB) larger than the 1 MiB staging slots: slots grow
    got = api._host_pair(tfb.Method.TWOFOLD_RIGOROUS, torch.from_numpy(xh), torch.from_numpy(yh), dev,
                         leaf_log2=21, engine=eng)
    _same(got, oracle.emulate(3, xh, yh, 21), "leaf larger than a slot")
    with pytest.raises(ValueError):  # mixed host/device operands are refused by the engine
        lib = _lib.lib()
        p = np.empty(2)
        _lib.check(lib.tf_host_reduce(eng, 2, 1, xt.data_ptr(), torch.from_numpy(yh[:8]).cuda().data_ptr(), 8, 0,
                                      p.ctypes.data, None))


def test_shards_form_subtrees_of_single_gpu_tree(tfb, oracle, cuda):
    """G shards reduced separately + tf_merge_tree == one-GPU result (power-of-two layout)."""
    n = 1 << 22
    x = tfb.philox_fill("uniform_sym", n, seed=4, stream=0)
    y = tfb.philox_fill("uniform_sym", n, seed=4, stream=1)
    lg = tfb.leaf_log2_for(torch.float64, n)
    for meth in tfb.Method:
        if meth is tfb.Method.WIDE:
            continue
        whole = tfb.reduce(meth, x, y).cpu()
        for G in (2, 4, 8):
            pairs = []
            for r in range(G):
                a, b = tfb.shard_range(n, r, G, lg)
                pairs.append(tfb.reduce(meth, x[a:b], y[a:b], leaf_log2=lg))
            merged = tfb.merge_pairs(meth, torch.stack(pairs)).cpu()
            assert torch.equal(merged, whole), (meth, G)
            # sharded_reduce on one process (world size 1 per shard call) agrees too
        assert torch.equal(tfb.sharded_reduce(meth, x, y, n_global=n).cpu(), whole)


def test_merge_tree_matches_oracle(tfb, oracle, cuda):
    rng = np.random.default_rng(5)
    for cnt in (0, 1, 2, 3, 7, 8, 255, 256, 257, 1000, 70_000):
        s = rng.standard_normal(cnt) * 1e3
        e = rng.standard_normal(cnt) * 1e-13
        pairs = torch.from_numpy(np.stack([s, e], 1)).to(cuda)
        for m in (0, 2, 3, 4):
            got = tfb.merge_pairs(list(tfb.Method)[m], pairs).cpu().numpy()
            _same(got, oracle.tree(m, np.float64, s, e), (cnt, m))


def test_philox_device_matches_host_twin(tfb, oracle, cuda):
    for dist in ("uniform01", "uniform_sym"):
        for dt, tdt in ((np.float32, torch.float32), (np.float64, torch.float64)):
            for off in (0, 12345, (1 << 32) + 7):
                d = tfb.philox_fill(dist, 4099, seed=9, stream=3, offset=off, dtype=tdt).cpu().numpy()
                h = oracle.philox_fill(dist, 4099, 9, 3, off, dt)
                assert d.tobytes() == h.tobytes(), (dist, dt, off)
    tot = 1 << 16
    for off, cnt in ((0, tot), (1000, 5000)):
        d = tfb.philox_fill("illcond", cnt, seed=2, offset=off, total=tot).cpu().numpy()
        h = oracle.philox_fill("illcond", cnt, 2, 0, off, np.float64, total=tot)
        assert d.tobytes() == h.tobytes()


def test_eft_kernels_known_answers(tfb):
    E = 2.0 ** -53
    assert tfb.fast_two_sum(1.0, 1.0) == (2.0, 0.0)
    assert tfb.fast_two_sum(1.0, E) == (1.0, E)
    assert tfb.fast_two_sum(2.0 ** 53, 1.0) == (2.0 ** 53, 1.0)
    for v in (0.5, -3.25, 1e300, 5e-324):
        assert tfb.two_sum(0.0, v) == (v, 0.0)
    assert tfb.two_sum(E, 1.0) == (1.0, E)
    x, y = tfb.two_sum(np.float32(1.0), np.float32(2.0 ** -24))
    assert isinstance(x, np.float32) and y == np.float32(2.0 ** -24)
    rng = np.random.default_rng(2024)
    a = (rng.uniform(-1, 1, 100_000) * 2.0 ** rng.integers(-20, 20, 100_000)).astype(np.float32)
    b = (rng.uniform(-1, 1, 100_000) * 2.0 ** rng.integers(-20, 20, 100_000)).astype(np.float32)
    x, y = tfb.two_sum(a, b)
    assert np.array_equal(x.astype(np.float64) + y.astype(np.float64), a.astype(np.float64) + b.astype(np.float64))
    x, y = tfb.two_sum(np.array([5e-324, 2e-308]), np.array([5e-324, -5e-324]))  # subnormals stay exact
    assert x[0] == 1e-323 and y[0] == 0.0


def test_errors_match_reference(tfb, cuda):
    with pytest.raises(TypeError):
        tfb.sum_wide(np.array([1.0]))
    with pytest.raises(TypeError):
        tfb.dot_direct(np.ones(3, np.float32), np.ones(3))
    with pytest.raises(ValueError):
        tfb.dot_direct(np.ones(3), np.ones(4))
    with pytest.raises(TypeError):
        tfb.sum_direct(np.arange(4))
    assert tfb.sum_twofold_fast(np.array([], np.float64)).twofold == (0.0, 0.0)
    r = tfb.sum_twofold_fast(np.array([3.5]))
    assert r.twofold == (3.5, 0.0)
    assert isinstance(tfb.sum_twofold_fast(np.ones(10, np.float32)).error, np.float32)
    assert isinstance(tfb.sum_wide(np.ones(10, np.float32)).value, np.float64)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_exact_integer_data_all_flavors(tfb, dt):
    """test_kernels.py:189-200 on every GPU flavor."""
    x = np.arange(1, 101, dtype=dt)
    for meth in tfb.Method:
        if meth is tfb.Method.WIDE and dt is not np.float32:
            continue
        for fl in (tfb.Flavor.sequential(), tfb.Flavor.unrolled(2), tfb.Flavor.unrolled(16),
                   tfb.Flavor.vectorized(4), tfb.Flavor.cuda()):
            r = tfb.run_flavor(meth, fl, x)
            assert float(r.value) == 5050.0 and float(r.error) == 0.0, (meth, fl)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_two_product_dot(tfb, oracle, cuda, dt):
    """Opt-in TwoProduct (TF_TRACK_PRODUCT): bit-exact with the emulator in every flavor,
    and v+e tracks the exact dot of the TRUE products (rigorous: to ~N eps^2)."""
    for n in (1, 17, 4097, 100_003, (1 << 20) + 3):
        xh = oracle.lcg_fill("mmix", n, 31, dt, True)
        yh = oracle.lcg_fill("nr", n, 32, dt, True)
        x, y = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
        for base, m in ((tfb.Method.TWOFOLD_FAST, 5), (tfb.Method.TWOFOLD_RIGOROUS, 6)):
            got = tfb.reduce(base, x, y, track_product=True).cpu().numpy()
            _same(got, oracle.emulate(m, xh, yh), (dt, n, m))
            if n <= 5000:
                for fl, want in ((tfb.Flavor.sequential(), oracle.seq(m, xh, yh)),
                                 (tfb.Flavor.unrolled(4), oracle.lanes(m, xh, yh, 4))):
                    _same(tfb.reduce(base, x, y, flavor=fl, track_product=True).cpu().numpy(), want, (fl, m))
        if n >= 4097:
            S, A = oracle.exact_true_dot(xh, yh), oracle.abs_true_dot(xh, yh)
            r = tfb.dot_twofold_rigorous(x, y, track_product=True)
            assert oracle.deviation(r.value, r.error, S) <= oracle.bound(3, dt, n, A)
    with pytest.raises(ValueError):
        tfb.reduce(tfb.Method.KAHAN, x, y, track_product=True)
    with pytest.raises(ValueError):
        tfb.reduce(tfb.Method.TWOFOLD_FAST, x, track_product=True)


def test_device_lcg_fill_matches_reference_fill(tfb, oracle, golden):
    """tf_lcg_fill == lcg.fill bit for bit (golden sha256 of the reference's own
    arrays), for whole arrays and arbitrary slices (jump-ahead)."""
    from golden_inputs import sha
    for key, pin in golden["lcg"].items():
        kind, dt, interval = key.split("_")
        tdt = torch.float32 if dt == "f32" else torch.float64
        d = tfb.lcg_fill(kind, pin["n"], pin["seed"], tdt, interval == "sym").cpu().numpy()
        assert sha(d) == pin["sha256"], key
    for kind in ("nr", "mmix"):
        for tdt, ndt in ((torch.float32, np.float32), (torch.float64, np.float64)):
            full = oracle.lcg_fill(kind, 200_000, 7, ndt, True)
            for off, cnt in ((0, 200_000), (1, 99), (12_345, 100_000), (199_990, 10)):
                d = tfb.lcg_fill(kind, cnt, 7, tdt, True, offset=off).cpu().numpy()
                assert d.tobytes() == full[off:off + cnt].tobytes(), (kind, tdt, off)


def test_gpu_exact_sum_matches_expansion_oracle(tfb, oracle, golden, cuda):
    """tf_exact == the reference's exact_sum (golden components) and the C
    expansion oracle, as rationals; hi/lo are the correctly rounded leading parts."""
    from fractions import Fraction
    inputs = load_inputs(oracle, golden)
    for name, rec in golden["inputs"].items():
        x, y = inputs[name]
        ref = sum((Fraction(float.fromhex(c)) for c in rec["exact"]), Fraction(0))
        # the fixture's dot oracle is over the kernels' addends (products rounded in the data type)
        got = tfb.exact_sum(x) if y is None else tfb.exact_dot(x, y, rounded_products=True)
        assert got.fraction() == ref, name
        assert got.hi == float(ref) if ref else got.hi == 0.0
        if ref:
            assert got.lo == float(ref - Fraction(got.hi)), name


def test_gpu_exact_hard_cases(tfb, oracle, cuda):
    from fractions import Fraction
    rng = np.random.default_rng(3)
    cases = [
        np.array([5e-324, 5e-324, -1e-320, 2.0 ** -1022]),            # subnormals
        np.array([1e308, -1e308, 1e-308, 3.0, -3.0]),                 # extreme exponents
        np.array([2.0 ** 53, 1.0, -(2.0 ** 53), 2.0 ** -60]),         # ties / cancellation
        rng.standard_normal(100_003) * 2.0 ** rng.integers(-600, 600, 100_003),
        oracle.philox_fill("illcond", 1 << 20, 2, 0, total=1 << 20),  # cfg3 layout
    ]
    for x in cases:
        want = sum((Fraction(float(v)) for v in x), Fraction(0)) if len(x) < 1000 else oracle.exact(x)
        got = tfb.exact_sum(x)
        assert got.fraction() == want
        assert got.hi == float(want)
        a = tfb.exact_sum(x, absolute=True)
        assert a.fraction() == (sum((abs(Fraction(float(v))) for v in x), Fraction(0)) if len(x) < 1000
                                else oracle.abs_sum(x))
    xf = oracle.lcg_fill("mmix", 300_001, 4, np.float32, True)
    yf = oracle.lcg_fill("nr", 300_001, 5, np.float32, True)
    assert tfb.exact_dot(xf, yf, rounded_products=True).fraction() == oracle.exact(xf, yf)
    assert tfb.exact_dot(xf, yf, true_products=True).fraction() == oracle.exact_true_dot(xf, yf)
    # default = expansion.exact_dot (expansion.py:112-126): binary32 sums the exact products
    assert tfb.exact_dot(xf, yf).fraction() == oracle.exact_true_dot(xf, yf)
    xd = oracle.lcg_fill("mmix", 300_001, 4, np.float64, True)
    yd = oracle.lcg_fill("nr", 300_001, 5, np.float64, True)
    assert tfb.exact_dot(xd, yd, true_products=True).fraction() == oracle.exact_true_dot(xd, yd)
    assert tfb.exact_dot(xd, yd).fraction() == oracle.exact(xd, yd)  # binary64: rounded products
    assert np.isnan(tfb.exact_sum(np.array([1.0, np.inf])).hi)
    # grid independence: a slice reduced in place == its copy
    xt = torch.from_numpy(xd).to(cuda)
    assert tfb.exact_sum(xt[1:]).fraction() == tfb.exact_sum(xt[1:].clone()).fraction()


def test_gpu_exact_hi_lo_random_signs_and_scales(tfb, cuda):
    """The warp-parallel finish (carry rounds, sign/magnitude, both roundings): hi = fl(S)
    and lo = fl(S - hi) exactly, against Fraction arithmetic, for totals of both signs,
    exact totals, totals that round up, cancellations to zero and overflow to inf."""
    from fractions import Fraction
    rng = np.random.default_rng(11)

    def check(x):
        want = sum((Fraction(float(v)) for v in x), Fraction(0))
        got = tfb.exact_sum(x)
        assert got.fraction() == want
        if want == 0:
            assert got.hi == 0.0 and got.lo == 0.0
            return
        hi = float(want)  # correctly rounded (Python's Fraction -> float rounds to nearest even)
        assert got.hi == hi, (x, got)
        assert got.lo == float(want - Fraction(hi)), (x, got)

    for _ in range(150):
        m = int(rng.integers(1, 40))
        x = rng.standard_normal(m) * 2.0 ** rng.integers(-1070, 1000, m)
        check(x)
        check(-x)
        check(np.concatenate([x, -x[: m // 2]]))
    check(np.array([1.0, -1.0, 2.0 ** -1074, -(2.0 ** -1074)]))  # exact zero
    check(np.array([2.0 ** 53, 1.0, 1.0]))                         # rounds up, lo negative
    check(np.array([-(2.0 ** 53), -1.0, -1.0]))
    check(np.array([2.0 ** 53, 1.0, 2.0 ** -60]))                  # above the tie: rounds up
    check(np.array([1.5, 2.0 ** -1074]))                           # lo subnormal
    big = tfb.exact_sum(np.array([1.7e308, 1.7e308]))
    assert big.hi == np.inf and big.lo == 0.0
    neg = tfb.exact_sum(np.array([-1.7e308, -1.7e308]))
    assert neg.hi == -np.inf


def test_cfg5_accuracy_at_full_scale_on_gpu(tfb, cuda):
    """BASELINE cfg5 (f64 dottf, N=2^32) is too large for the CPU oracle in a test;
    the GPU exact dot checks the twofold result at full size (64 GiB resident)."""
    from fractions import Fraction
    free, _ = torch.cuda.mem_get_info()
    n = 1 << 32 if free > 80 * 2**30 else 1 << 30
    x = tfb.philox_fill("uniform_sym", n, seed=4, stream=0)
    y = tfb.philox_fill("uniform_sym", n, seed=4, stream=1)
    r = tfb.dot_twofold_fast(x, y)
    S = tfb.exact_dot(x, y).fraction()
    A = tfb.exact_dot(x, y, absolute=True).fraction()
    eps = Fraction(2.0 ** -53)
    D = abs(Fraction(float(r.value)) + Fraction(float(r.error)) - S)
    assert D <= 2 * n * eps * eps * A + Fraction(1, 64) * eps * A
    rr = tfb.dot_twofold_rigorous(x, y)
    assert abs(Fraction(float(rr.value)) + Fraction(float(rr.error)) - S) <= 2 * n * eps * eps * A
    del x, y
    torch.cuda.empty_cache()


def test_leaf_split_is_result_neutral(tfb, oracle, cuda):
    """Splitting leaves over 1/2/4 CTAs (grid balance) never changes a bit."""
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    try:
        for dt in (np.float32, np.float64):
            for n in (5, 4097, 100_003, 1 << 20, (1 << 22) + 9):
                xh = oracle.lcg_fill("mmix", n, 41, dt, True)
                yh = oracle.lcg_fill("nr", n, 42, dt, True)
                x, y = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
                for m in _methods(dt):
                    meth = list(tfb.Method)[m]
                    want = oracle.emulate(m, xh, yh)
                    for split in (1, 2, 4):
                        assert L.tf_set_leaf_split(split) == 0
                        _same(tfb.reduce(meth, x, y).cpu().numpy(), want, (dt, n, m, split))
                X = torch.from_numpy(oracle.lcg_fill("nr", 37 * 5000, 43, dt, True).reshape(37, 5000)).to(cuda)
                ref = None
                for split in (1, 2, 4):
                    L.tf_set_leaf_split(split)
                    got = tfb.reduce_rows(tfb.Method.TWOFOLD_RIGOROUS, X).cpu()
                    ref = got if ref is None else ref
                    assert torch.equal(got, ref)
    finally:
        L.tf_set_leaf_split(0)


def test_tma_loader_bit_identical(tfb, oracle, cuda):
    """The bulk-copy (TMA engine) pipeline loader gives the same bits as the LDG loader
    and the emulator: full and partial leaves, sums, dots, rows."""
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    try:
        for dt in (np.float32, np.float64):
            for n in (17, 4097, 100_003, (1 << 21) + 9):
                xh = oracle.lcg_fill("mmix", n, 51, dt, True)
                yh = oracle.lcg_fill("nr", n, 52, dt, True)
                x, y = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
                for m in _methods(dt):
                    meth = list(tfb.Method)[m]
                    for yy, yyh in ((None, None), (y, yh)):
                        want = oracle.emulate(m, xh, yyh)
                        for loader in (1, 2, 3, 6, 7):
                            assert L.tf_set_loader(loader) == 0
                            _same(tfb.reduce(meth, x, yy).cpu().numpy(), want, (dt, n, m, loader))
            X = tfb.rows_scaled_normal(33, 70_000, seed=5, stream=0, dtype=torch.float32)
            Y = tfb.rows_scaled_normal(33, 70_000, seed=5, stream=1, dtype=torch.float32)
            L.tf_set_loader(1)
            ref = tfb.reduce_rows(tfb.Method.TWOFOLD_FAST, X, Y).cpu()
            for loader in (0, 2, 3, 6, 7):
                L.tf_set_loader(loader)
                assert torch.equal(tfb.reduce_rows(tfb.Method.TWOFOLD_FAST, X, Y).cpu(), ref)
    finally:
        L.tf_set_loader(0)


def test_pdl_tail_bit_identical(tfb, oracle, cuda):
    """Partials-only launch + programmatic-dependent tree kernel == the fused
    single launch == the emulator (also with leaf splits)."""
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    try:
        for dt in (np.float32, np.float64):
            for n in (17, 70_001, (1 << 21) + 9):
                xh = oracle.lcg_fill("mmix", n, 61, dt, True)
                yh = oracle.lcg_fill("nr", n, 62, dt, True)
                x, y = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
                for m in _methods(dt):
                    meth = list(tfb.Method)[m]
                    want = oracle.emulate(m, xh, yh)
                    for split in (1, 2):
                        L.tf_set_leaf_split(split)
                        L.tf_set_tail(2)
                        _same(tfb.reduce(meth, x, y).cpu().numpy(), want, (dt, n, m, split))
        X = tfb.rows_scaled_normal(37, 70_000, seed=6, stream=0, dtype=torch.float32)
        L.tf_set_tail(1)
        L.tf_set_leaf_split(1)
        ref = tfb.reduce_rows(tfb.Method.TWOFOLD_RIGOROUS, X).cpu()
        L.tf_set_tail(2)
        assert torch.equal(tfb.reduce_rows(tfb.Method.TWOFOLD_RIGOROUS, X).cpu(), ref)
    finally:
        L.tf_set_tail(0)
        L.tf_set_leaf_split(0)


def test_small_cluster_path_bit_identical(tfb, oracle, cuda):
    """Single-cluster small path (<= 64 one-vector leaves, small.cuh) == emulator ==
    PDL / ticket tails: every method, dtype, sum/dot, ragged sizes across every
    cluster size (1..16 CTAs), 16-byte-misaligned (scalar) inputs, TwoProduct."""
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    try:
        for dt in (np.float32, np.float64):
            V = 4 if dt == np.float32 else 2
            leaf = 256 * V
            for n in (1, 5, leaf - 1, leaf, leaf + 3, 3 * leaf, 4 * leaf + 1, 9 * leaf - 7, 33 * leaf, 64 * leaf):
                xh = oracle.lcg_fill("mmix", n + 1, 71, dt, True)
                yh = oracle.lcg_fill("nr", n + 1, 72, dt, True)
                xd, yd = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)
                for off in (0, 1):  # off = 1: misaligned views take the scalar path
                    x, y = xd[off:off + n], yd[off:off + n]
                    xs, ys = xh[off:off + n], yh[off:off + n]
                    for m in _methods(dt):
                        meth = list(tfb.Method)[m]
                        for dot in (False, True):
                            want = oracle.emulate(m, xs, ys if dot else None)
                            L.tf_set_tail(0)
                            got = tfb.reduce(meth, x, y if dot else None).cpu().numpy()
                            assert "small_cluster_kernel" in L.tf_last_launch().decode()
                            _same(got, want, (dt, n, off, m, dot))
                            for tail in (1, 2):
                                L.tf_set_tail(tail)
                                _same(tfb.reduce(meth, x, y if dot else None).cpu().numpy(), want,
                                      (dt, n, off, m, dot, tail))
                    L.tf_set_tail(0)
                    for meth in (tfb.Method.TWOFOLD_FAST, tfb.Method.TWOFOLD_RIGOROUS):
                        got = tfb.reduce(meth, x, y, track_product=True).cpu().numpy()
                        L.tf_set_tail(2)
                        _same(got, tfb.reduce(meth, x, y, track_product=True).cpu().numpy(), (dt, n, off, "tp"))
                        L.tf_set_tail(0)
    finally:
        L.tf_set_tail(0)


def test_gpu_exact_near_overflow(tfb, cuda):
    """Partial sums beyond binary64 range stay exact in the superaccumulator."""
    from fractions import Fraction
    for x in (np.array([1e308, 1e308, -1e308, 5.0]), np.full(1000, 1.7e308), np.array([1e308] * 7 + [-1e308] * 7 + [1.0])):
        got = tfb.exact_sum(x)
        want = sum((Fraction(float(v)) for v in x), Fraction(0))
        assert got.fraction() == want
        assert got.hi == (float(want) if abs(want) < Fraction(2) ** 1024 else (np.inf if want > 0 else -np.inf))


def test_blocking_wrappers_order_after_the_current_stream(tfb, oracle, cuda):
    """run_flavor on CUDA tensors goes through tf_host_reduce on the engine's own
    stream; it must start after the work pending on the caller's stream."""
    n = 1 << 24
    x = torch.zeros(n, dtype=torch.float32, device=cuda)
    for _ in range(20):  # a queue of pending writes on the default stream
        x.add_(0.5)
    r = tfb.sum_twofold_fast(x)
    assert float(r.value) + float(r.error) == 10.0 * n
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y = torch.empty(n, dtype=torch.float64, device=cuda)
        y.fill_(2.0)
        for _ in range(10):
            y.mul_(1.5)
        r = tfb.dot_twofold_rigorous(y, y)
    assert float(r.value) == n * (2.0 * 1.5 ** 10) ** 2
    xh = oracle.lcg_fill("mmix", 70_001, 81, np.float64, True)
    xd = torch.from_numpy(xh).to(cuda)
    r = tfb.sum_twofold_fast(xd)
    _same((r.value, r.error), oracle.emulate(2, xh), "device tensor wrapper")


def test_thread_safety_many_streams(tfb, oracle, cuda):
    """The reference's functions are pure and thread-safe: several host
    threads, each on its own CUDA stream (own scratch) plus the shared host engine,
    get bit-identical results to a single-threaded run."""
    import threading
    sizes = (5_001, 70_001, (1 << 20) + 3)
    data = {}
    for n in sizes:
        xh = oracle.lcg_fill("mmix", n, 91, np.float64, True)
        yh = oracle.lcg_fill("nr", n, 92, np.float64, True)
        data[n] = (xh, yh, torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda), oracle.emulate(2, xh, yh))
    errors = []

    def worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for it in range(40):
                    n = sizes[(k + it) % len(sizes)]
                    xh, yh, xd, yd, want = data[n]
                    got = tfb.reduce(tfb.Method.TWOFOLD_FAST, xd, yd).cpu().numpy()
                    assert float(got[0]).hex() == float(want[0]).hex() and float(got[1]).hex() == float(want[1]).hex()
                    r = tfb.dot_twofold_fast(xh, yh)  # numpy: the shared host engine
                    assert float(r.value).hex() == float(want[0]).hex() and float(r.error).hex() == float(want[1]).hex()
        except Exception as exc:  # surfaced in the main thread
            errors.append(repr(exc))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:3]


def _same_nf(got, want, ctx):
    """Bit-exact, except that every NaN matches every NaN (payload/sign of a
    generated NaN is implementation-defined: x86 0xFFF8..., CUDA 0x7FFF...)."""
    for g, w in zip((float(got[0]), float(got[1])), (float(want[0]), float(want[1]))):
        if np.isnan(w):
            assert np.isnan(g), (ctx, got, want)
        else:
            assert g.hex() == w.hex(), (ctx, got, want)


def test_non_finite_inputs_grid_and_seq(tfb, oracle, cuda):
    """inf / -inf / NaN addends and overflowing products propagate exactly as in the
    reference recurrence (seq flavor vs the oracle's restatement) and as in the
    GPU tree (grid flavor vs the emulator), for every method."""
    rng = np.random.default_rng(7)
    for dt in (np.float32, np.float64):
        big = np.finfo(dt).max
        for n in (37, 5_001, 200_003):
            base = rng.uniform(-1, 1, n).astype(dt)
            cases = []
            for pat in ("inf", "ninf", "both", "nan", "ovf"):
                x = base.copy()
                y = rng.uniform(-1, 1, n).astype(dt)
                if pat == "inf":
                    x[n // 3] = np.inf
                elif pat == "ninf":
                    x[n // 2] = -np.inf
                elif pat == "both":
                    x[1], x[n - 2] = np.inf, -np.inf
                elif pat == "nan":
                    x[n // 5] = np.nan
                else:  # finite inputs whose sum / products overflow
                    x[:4] = big
                    y[:4] = dt(4)
                cases.append((pat, x, y))
            for pat, x, y in cases:
                xd, yd = torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda)
                for m in _methods(dt):
                    meth = list(tfb.Method)[m]
                    for dot in (False, True):
                        yy, yyh = (yd, y) if dot else (None, None)
                        _same_nf(tfb.reduce(meth, xd, yy).cpu().numpy(), oracle.emulate(m, x, yyh),
                                 (dt, n, pat, m, dot, "grid"))
                        if n <= 5_001:
                            seq = tfb.reduce(meth, xd, yy, flavor=tfb.Flavor.sequential()).cpu().numpy()
                            _same_nf(seq, oracle.seq(m, x, yyh), (dt, n, pat, m, dot, "seq"))


def test_wrappers_accept_strided_numpy_lists_and_views(tfb, oracle, cuda):
    """kernels.py:575 copies non-contiguous inputs (np.ascontiguousarray): strided
    numpy views, Python lists and CPU tensors give the contiguous array's result."""
    base = oracle.lcg_fill("mmix", 20_002, 111, np.float64, True)
    view = base[::2]
    want = oracle.emulate(2, np.ascontiguousarray(view))
    for arg in (view, list(view), torch.from_numpy(base)[::2]):
        r = tfb.sum_twofold_fast(arg)
        assert _hex(r.value) == _hex(want[0]) and _hex(r.error) == _hex(want[1]), type(arg)
    f32 = base.astype(np.float32)
    r = tfb.sum_wide(f32[1::3])
    w = oracle.emulate(1, np.ascontiguousarray(f32[1::3]))
    assert _hex(r.value) == _hex(w[0]) and type(r.value) is np.float64


def test_host_rows_engine_equals_device_rows(tfb, oracle, cuda):
    """tf_host_reduce_rows (row blocks staged + overlapped, pitched DMA for pinned strided
    input) == tf_reduce_rows on the device copy, bit for bit; many blocks via 1 MiB slots.
    Rows longer than a slot (300_001 f64 / 600_001 f32 elements > 1 MiB) stream through
    leaf-aligned chunks one row at a time (never size the slots to a whole row)."""
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    eng = _lib.host_engine(0, chunk_bytes=1 << 20, threads=3)
    for dt, code in ((np.float32, 0), (np.float64, 1)):
        long_cols = 300_001 if dt == np.float64 else 600_001
        for rows, cols, ld in ((37, 70_001, 70_001), (9, 4_999, 5_000), (300, 1_000, 1_003), (2, 3, 3),
                               (3, long_cols, long_cols), (3, long_cols, long_cols + 3)):
            base = oracle.lcg_fill("mmix", rows * ld, 121, dt, True).reshape(rows, ld)
            ybase = oracle.lcg_fill("nr", rows * ld, 122, dt, True).reshape(rows, ld)
            want = {}
            for m in (0, 2, 3, 4):
                meth = list(tfb.Method)[m]
                xd = torch.from_numpy(base).to(cuda)[:, :cols]
                yd = torch.from_numpy(ybase).to(cuda)[:, :cols]
                want[m] = tfb.reduce_rows(meth, xd, yd).cpu().numpy()
            for pinned in (False, True):
                xt = torch.from_numpy(base)
                yt = torch.from_numpy(ybase)
                if pinned:
                    xt, yt = xt.pin_memory(), yt.pin_memory()
                xs, ys = xt[:, :cols], yt[:, :cols]
                for m in (0, 2, 3, 4):
                    out = np.empty((rows, 2), dt)
                    rc = L.tf_host_reduce_rows(eng, m, code, xs.data_ptr(), ys.data_ptr(), rows, cols, ld, ld, 0,
                                               out.ctypes.data, None)
                    assert rc == 0, L.tf_strerror(rc)
                    assert np.array_equal(out.view(np.uint8), want[m].view(np.uint8)), (dt, rows, cols, ld, pinned, m)
                    # and through the public API (default engine)
                    got = tfb.reduce_rows(list(tfb.Method)[m], xs, ys).cpu().numpy()
                    assert np.array_equal(got.view(np.uint8), want[m].view(np.uint8)), (dt, rows, cols, "api")


def test_non_finite_rows_every_rows_kernel(tfb, oracle, cuda):
    """inf / -inf / NaN and overflowing entries in row-wise reductions: the lane-group kernel
    (aligned, 32-byte and misaligned-select loads) and the CTA-per-row kernel propagate them
    exactly as the emulator's per-row tree (NaN payloads excepted)."""
    L = tfb._lib.lib()
    rng = np.random.default_rng(8)
    try:
        for dt in (np.float32, np.float64):
            big = np.finfo(dt).max
            for rows, cols, pad in ((40, 64, 0), (33, 1000, 0), (29, 63, 1), (17, 300, 3)):
                ld = cols + pad
                X = rng.uniform(-1, 1, (rows, ld)).astype(dt)
                Y = rng.uniform(-1, 1, (rows, ld)).astype(dt)
                X[1, cols // 2] = np.inf
                X[2, 0], X[2, cols - 1] = np.inf, -np.inf
                X[3, cols // 3] = np.nan
                X[4, :2], Y[4, :2] = big, dt(4)
                Xd = torch.from_numpy(X).to(cuda)[:, :cols]
                Yd = torch.from_numpy(Y).to(cuda)[:, :cols]
                Xh, Yh = np.ascontiguousarray(X[:, :cols]), np.ascontiguousarray(Y[:, :cols])
                for m in _methods(dt):
                    meth = list(tfb.Method)[m]
                    ev, ee = oracle.emulate_rows(m, Xh, Yh)
                    for kind in (1, 2):
                        L.tf_set_rows_kernel(kind)
                        got = tfb.reduce_rows(meth, Xd, Yd).cpu().numpy()
                        for r in range(rows):
                            _same_nf(got[r], (ev[r], ee[r]), (dt, rows, cols, pad, m, kind, r))
    finally:
        L.tf_set_rows_kernel(0)


def test_non_finite_misaligned_views(tfb, oracle, cuda):
    """Non-finite entries through the misaligned paths (binary32 shifted-vector loads,
    binary64 batched element loads), vs the emulator (NaN payloads excepted)."""
    rng = np.random.default_rng(9)
    for dt in (np.float32, np.float64):
        n = 300_001
        for off in (1, 2, 3) if dt == np.float32 else (1,):
            x = rng.uniform(-1, 1, n + 4).astype(dt)
            y = rng.uniform(-1, 1, n + 4).astype(dt)
            x[off + 1000] = np.inf
            x[off + 200_000] = -np.inf if off % 2 else np.nan
            xd, yd = torch.from_numpy(x).to(cuda), torch.from_numpy(y).to(cuda)
            xs, ys = x[off:off + n], y[off:off + n]
            for m in _methods(dt):
                meth = list(tfb.Method)[m]
                got = tfb.reduce(meth, xd[off:off + n], yd[off:off + n]).cpu().numpy()
                _same_nf(got, oracle.emulate(m, xs, ys), (dt, off, m))


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_rows_class_uniform_kernel_matches_emulator(tfb, oracle, cuda, dt):
    """Misaligned pitches on the class-uniform warps (rows_cls_kernel: rows of one 32-byte
    offset class per warp, 32-byte windows, compile-time element picks) == the emulator's
    per-row tree, for every offset class, partial last blocks, sums and dots, and several
    periods (pitch mod 32 bytes); x / y on different class sequences take the select path."""
    L = tfb._lib.lib()
    item = np.dtype(dt).itemsize
    for cols, pad, off in ((777, 0, 1), (255, 2, 3), (17, 0, 1), (63, 1, 2), (1001, 0, 0), (130, 3, 1)):
        rows = 203
        ld = cols + pad
        if (ld * item) % 16 == 0 and off * item % 16 == 0:
            continue  # aligned: not this kernel
        bx = oracle.lcg_fill("mmix", rows * ld + 8, 71 + cols, dt, True)
        by = oracle.lcg_fill("nr", rows * ld + 8, 72 + cols, dt, True)
        bx[5 * ld + 3] = -0.0
        X = torch.from_numpy(bx).to(cuda)[off:off + rows * ld].view(rows, ld)[:, :cols]
        Y = torch.from_numpy(by).to(cuda)[off:off + rows * ld].view(rows, ld)[:, :cols]
        Xh, Yh = np.ascontiguousarray(X.cpu().numpy()), np.ascontiguousarray(Y.cpu().numpy())
        for m in _methods(dt):
            meth = list(tfb.Method)[m]
            for yy, yyh in ((None, None), (Y, Yh)):
                got = tfb.reduce_rows(meth, X, yy).cpu().numpy()
                desc = L.tf_last_launch().decode()
                if cols <= 1024 and cols * item > 128:  # one-lane rows (<= 8 vectors) keep element loads
                    assert "rows_cls_kernel" in desc, desc
                ev, ee = oracle.emulate_rows(m, Xh, yyh)
                for r in range(rows):
                    _same(got[r], (ev[r], ee[r]), (dt, cols, pad, off, m, r, yy is None))
        # y on another class sequence (offset differs by one element): the select path, same bits
        Y2 = torch.from_numpy(by).to(cuda)[off + 1:off + 1 + rows * ld].view(rows, ld)[:, :cols]
        Y2h = np.ascontiguousarray(Y2.cpu().numpy())
        got = tfb.reduce_rows(tfb.Method.TWOFOLD_FAST, X, Y2).cpu().numpy()
        assert "rows_cls_kernel" not in L.tf_last_launch().decode()
        ev, ee = oracle.emulate_rows(2, Xh, Y2h)
        for r in range(rows):
            _same(got[r], (ev[r], ee[r]), (dt, cols, "y other class", r))

@pytest.mark.gpu
def test_prefetch_preamble_is_result_neutral(tfb, oracle, cuda):
    """The L2 prefetch preamble of the leaves / single-cluster kernels (tf_set_prefetch: off,
    automatic, 4 KiB .. 512 KiB per operand per CTA) never changes a bit: ragged sizes whose
    last leaf is partial or not a multiple of 16 bytes, rows with a padded pitch, sums and
    dots, back-to-back launches in one stream (the preamble runs while the previous call's
    tree kernel retires), inputs ending exactly at the end of their allocation."""
    from paper_1401_0248_b200 import _lib
    L = _lib.lib()
    assert L.tf_set_prefetch(-2) == _lib.TF_EINVAL_ARG and L.tf_set_prefetch(513) == _lib.TF_EINVAL_ARG
    try:
        for dt in (np.float32, np.float64):
            for n in (1023, 4096, 100003, (1 << 18) + 5, 1 << 20, (3 << 20) + 1234):
                xh = oracle.lcg_fill("mmix", n, 81, dt, True)
                yh = oracle.lcg_fill("nr", n, 82, dt, True)
                x, y = torch.from_numpy(xh).to(cuda), torch.from_numpy(yh).to(cuda)  # exact-size allocations
                for dot in (False, True):
                    want = oracle.emulate(2, xh, yh if dot else None)
                    for kb in (0, -1, 4, 32, 512):
                        assert L.tf_set_prefetch(kb) == 0
                        outs = [tfb.reduce(tfb.Method.TWOFOLD_FAST, x, y if dot else None) for _ in range(3)]
                        for o in outs:
                            _same(o.cpu().numpy(), want, (dt, n, dot, kb))
        rows, cols, ld = 7, 70001, 70016
        mh = oracle.lcg_fill("mmix", rows * ld, 83, np.float32, True).reshape(rows, ld)
        m = torch.from_numpy(mh).to(cuda)
        ev, ee = oracle.emulate_rows(3, mh[:, :cols], mh[:, :cols])
        for kb in (0, -1, 64, 512):
            L.tf_set_prefetch(kb)
            got = tfb.reduce_rows(tfb.Method.TWOFOLD_RIGOROUS, m[:, :cols], m[:, :cols]).cpu().numpy()
            for r in range(rows):
                _same(got[r], (ev[r], ee[r]), ("rows", kb, r))
    finally:
        L.tf_set_prefetch(-1)



