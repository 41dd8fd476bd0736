"""Host-side logic of the drop-in API (no GPU needed): mirrors test_kernels.py's
flavor/validation tests and the exception contract of kernels.py:574-601."""

import os
import re

import numpy as np
import pytest
import torch

import paper_1401_0248_b200 as tfb
from paper_1401_0248_b200 import Flavor, Method

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_method_enum_matches_reference():
    # kernels.py:44-49
    assert [m.value for m in Method] == ["direct", "wide", "twofold-fast", "twofold-rigorous", "kahan"]


def test_flavor_validation_like_reference():
    # test_kernels.py:243-251
    with pytest.raises(ValueError):
        Flavor.unrolled(3)
    with pytest.raises(ValueError):
        Flavor.vectorized(32)
    with pytest.raises(ValueError):
        Flavor.parse("turbo")
    assert Flavor.parse("unroll:4").lanes == 4
    assert str(Flavor.parse("vec:8")) == "vec:8"
    with pytest.raises(ValueError):
        Flavor("seq", 4)
    assert str(Flavor.parse("cuda")) == "cuda" and Flavor.parse("cuda") == Flavor.cuda()
    with pytest.raises(ValueError):
        Flavor.parse("cuda:4")
    assert str(Flavor.unrolled()) == "unroll" and str(Flavor.sequential()) == "seq"


def test_input_errors_raised_before_any_device_work():
    with pytest.raises(TypeError):
        tfb.sum_wide(np.array([1.0]))               # kernels.py:600-601
    with pytest.raises(TypeError):
        tfb.dot_direct(np.ones(3, np.float32), np.ones(3))   # :580-581
    with pytest.raises(ValueError):
        tfb.dot_direct(np.ones(3), np.ones(4))      # :582-583
    with pytest.raises(TypeError):
        tfb.sum_direct(np.arange(4))                # :576-577
    with pytest.raises(TypeError):
        tfb.sum_direct(torch.ones(4, dtype=torch.float16))
    with pytest.raises(ValueError):
        tfb.sum_direct(np.ones((2, 2)))
    with pytest.raises(TypeError):
        tfb.dot_rows(Method.TWOFOLD_FAST, np.ones((2, 3), np.float32), np.ones((2, 3)))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """Without a GPU the product fails loudly instead of computing on the CPU."""
    with pytest.raises(RuntimeError, match="no CUDA device"):
        tfb.sum_twofold_fast(np.ones(10))
    with pytest.raises(RuntimeError):
        tfb.run_flavor(Method.DIRECT, Flavor.sequential(), np.ones(10))


def test_product_never_touches_the_oracle():
    pkg = os.path.join(REPO, "paper_1401_0248_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(root, f)).read()
                # comments may cite the oracle; code may not import, include or load it
                assert not re.search(r"^\s*(import\s+oracle|from\s+oracle|#\s*include\s*[<\"].*oracle)|libtfo", src,
                                     flags=re.M), f


def test_leaf_rule_and_shard_ranges(oracle):
    for n in (1, 100, 1 << 20, 1 << 24, (1 << 29) * 8):
        for dt, odt in ((torch.float32, np.float32), (torch.float64, np.float64)):
            assert tfb.leaf_log2_for(dt, n) == oracle.leaf_log2_auto(odt, n)
    n = 1 << 32
    lg = tfb.leaf_log2_for(torch.float64, n)
    assert lg == 16
    for G in (1, 2, 4, 8):
        spans = [tfb.shard_range(n, r, G, lg) for r in range(G)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert all((b - a) == n // G and a % (1 << lg) == 0 for a, b in spans)
    # ragged: leaf-aligned, covering, as even as possible
    n, lg, G = 1_000_003, 12, 3
    spans = [tfb.shard_range(n, r, G, lg) for r in range(G)]
    assert spans[0][0] == 0 and spans[-1][1] == n and all(a % 4096 == 0 for a, _ in spans)
    with pytest.raises(ValueError):
        tfb.shard_range(10, 3, 3, 9)


def test_product_host_twin_matches_oracle_twin(oracle):
    """tf_fill_host (product, CPU) == the oracle's independent Philox restatement
    (and, in test_gpu_parity.py, == the device stream)."""
    for dist in ("uniform01", "uniform_sym"):
        for dt, ndt in ((torch.float32, np.float32), (torch.float64, np.float64)):
            a = tfb.philox_fill_host(dist, 100_003, seed=9, stream=3, offset=77, dtype=dt).numpy()
            b = oracle.philox_fill(dist, 100_003, 9, 3, 77, ndt)
            assert a.tobytes() == b.tobytes(), (dist, dt)
    a = tfb.philox_fill_host("illcond", 1 << 16, seed=2, total=1 << 16).numpy()
    b = oracle.philox_fill("illcond", 1 << 16, 2, 0, 0, np.float64, total=1 << 16)
    assert a.tobytes() == b.tobytes()
    with pytest.raises(ValueError):
        tfb.philox_fill_host("normal", 10, seed=1)
