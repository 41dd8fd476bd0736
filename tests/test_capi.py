"""The C-ABI library loads without a GPU and exports every symbol include/*.h declares."""

import ctypes
import os
import re

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "twofold_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(tf_\w+)\s*\(", src, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_1401_0248_b200 import _lib
    return _lib.lib()


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("tf_reduce", "tf_reduce_rows", "tf_reduce_leaves", "tf_merge_tree", "tf_reduce_seq",
                 "tf_reduce_lanes", "tf_eft", "tf_fill", "tf_fill_rows_scaled", "tf_canary", "tf_strerror",
                 "tf_workspace_size", "tf_leaf_log2", "tf_version", "tf_last_cuda_error"):
        assert must in names


def test_every_declared_symbol_is_exported(lib):
    raw = ctypes.CDLL(lib._name)
    for name in declared_functions():
        assert hasattr(raw, name), name


def test_host_only_entry_points(lib, oracle):
    from paper_1401_0248_b200 import _lib
    assert lib.tf_version() >= 1
    assert lib.tf_strerror(_lib.TF_EINVAL_DTYPE).decode().startswith("unsupported dtype")
    for dt in (0, 1):
        for n in (0, 1, 2, 1000, 1 << 16, (1 << 20) + 1, 1 << 24, 1 << 29, 1 << 32, 1 << 40):
            assert lib.tf_leaf_log2(dt, n) == oracle.lib().tfo_leaf_log2(dt, n), (dt, n)


def test_validation_before_any_device_work(lib):
    from paper_1401_0248_b200 import _lib
    # argument errors are reported without touching the GPU (none here)
    assert lib.tf_reduce(9, 0, None, None, 10, 0, None, None, 0, None, 0, None) == _lib.TF_EINVAL_METHOD
    assert lib.tf_reduce(1, 1, None, None, 10, 0, None, None, 0, None, 0, None) == _lib.TF_EINVAL_DTYPE
    assert lib.tf_reduce(2, 5, None, None, 10, 0, None, None, 0, None, 0, None) == _lib.TF_EINVAL_DTYPE
    assert lib.tf_reduce(2, 1, None, None, -1, 0, None, None, 0, None, 0, None) == _lib.TF_EINVAL_SHAPE
    assert lib.tf_reduce_lanes(2, 1, None, None, 8, 3, None, None) == _lib.TF_EINVAL_ARG
    assert lib.tf_reduce_lanes(2, 1, None, None, 8, 32, None, None) == _lib.TF_EINVAL_ARG
    assert lib.tf_reduce(2, 1, None, None, 10, 3, None, None, 0, None, 0, None) == _lib.TF_EINVAL_ARG
    assert lib.tf_fill(7, 1, 0, 0, 0, 10, 0, 0, 0, 0, None, None) == _lib.TF_EINVAL_ARG
    # multi-leaf input without scratch
    assert lib.tf_reduce(2, 1, 16, None, 1 << 20, 0, 16, None, 0, None, 0, None) == _lib.TF_EWORKSPACE


def test_workspace_size(lib):
    from paper_1401_0248_b200 import Method, workspace_size
    import torch
    pb, cnt, leaves = workspace_size(Method.TWOFOLD_FAST, torch.float64, 1, 1 << 29)
    # partials are sized for the largest leaf split (4 unit pairs per leaf)
    assert leaves == (1 << 29) >> 16 and pb == 4 * leaves * 16 and cnt == 1
    pb, cnt, leaves = workspace_size(Method.WIDE, torch.float32, 4096, 65536)
    assert leaves == 1 and pb == 0 and cnt == 0  # one leaf per row: pairs go straight to out
    pb, cnt, leaves = workspace_size(Method.WIDE, torch.float32, 4096, 65537)
    assert leaves == 2 and pb == 4 * 4096 * 2 * 16 and cnt == 4096  # wide pairs are binary64
    pb, cnt, leaves = workspace_size(Method.TWOFOLD_FAST, torch.float32, 1, 100)
    assert leaves == 1 and pb == 4 * 8 and cnt == 1  # 1-D: the pair slots stay (peer combine)
    pb, cnt, leaves = workspace_size(Method.KAHAN, torch.float32, 1, 1 << 24)
    assert leaves == (1 << 24) >> 15 and pb == 4 * leaves * 8


def test_host_engine_entry_points_without_gpu(lib):
    """The host-buffer engine validates its handle and fails cleanly with no device."""
    from paper_1401_0248_b200 import _lib
    out = ctypes.c_double * 2
    assert lib.tf_host_reduce(None, 2, 1, None, None, 0, 0, out(), None) == _lib.TF_EINVAL_ARG
    assert lib.tf_host_engine_destroy(None) == _lib.TF_OK
    assert lib.tf_host_engine_threads(None) == 0
    eng = ctypes.c_void_p()
    assert lib.tf_host_engine_create(0, 0, 0, None) == _lib.TF_EINVAL_ARG
    rc = lib.tf_host_engine_create(0, 0, 0, ctypes.byref(eng))
    if rc == _lib.TF_OK:  # a GPU is visible: clean up
        assert lib.tf_host_engine_threads(eng) >= 1
        assert lib.tf_host_engine_destroy(eng) == _lib.TF_OK
    else:
        assert rc in (_lib.TF_ECUDA, _lib.TF_EINVAL_ARG) and not eng.value


def test_first_host_engine_call_loads_the_library_without_deadlock():
    """host_engine() as the very first library call (lib() not loaded yet) must not
    self-deadlock on the loader lock; with no GPU it raises instead."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, %r)\n"
            "from paper_1401_0248_b200 import _lib\n"
            "try:\n    _lib.host_engine(0)\n    print('created')\n"
            "except RuntimeError as e:\n    print('raised', e)\n") % REPO
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.startswith(("created", "raised"))
