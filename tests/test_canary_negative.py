"""Negative control for the strict-rounding canary (test_acceptance.py:243-258).

The reference proves its canary can fail by compiling the same expression
with numba fastmath=True.  Here canary.cu is built a second time with plain
operators and --use_fast_math (csrc/Makefile: build/libtfb_canary_unsafe.so,
never loaded by the package): its SASS must contain a contracted FMA, its
tf_canary must return TF_ECANARY on the GPU, and the package's import-time
check must raise RuntimeError when handed such a canary.
"""

import ctypes
import os
import re
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNSAFE = os.path.join(REPO, "paper_1401_0248_b200", "csrc", "build", "libtfb_canary_unsafe.so")
PRODUCT = os.path.join(REPO, "paper_1401_0248_b200", "libtwofold_b200.so")


def _canary_sass(path):
    out = subprocess.run(["cuobjdump", "-sass", path], check=True, capture_output=True, text=True).stdout
    body, on = [], False
    for line in out.splitlines():
        if "Function :" in line:
            on = "canary_kernel" in line
        elif on:
            body.append(line)
    return "\n".join(body)


@pytest.mark.skipif(not shutil.which("cuobjdump"), reason="cuobjdump not installed")
def test_unsafe_build_contracts_and_product_does_not():
    assert os.path.exists(UNSAFE), "negative-control canary not built (make -C paper_1401_0248_b200/csrc)"
    unsafe = _canary_sass(UNSAFE)
    safe = _canary_sass(PRODUCT)
    assert unsafe and safe
    assert re.search(r"\b[DF]FMA\b", unsafe), "the fast-math canary build should contain a contracted FMA"
    assert not re.search(r"\b[DF]FMA\b|\.FTZ\b", safe), "the product canary must not contract or flush"


@pytest.mark.gpu
def test_canary_rejects_the_unsafe_build(cuda):
    from paper_1401_0248_b200 import _lib
    bad = ctypes.CDLL(UNSAFE)
    bad.tf_canary.restype = ctypes.c_int
    bad.tf_canary_raw.argtypes = [ctypes.POINTER(ctypes.c_double)]
    out = (ctypes.c_double * 8)()
    assert bad.tf_canary_raw(out) == _lib.TF_OK
    # fl(fl(a*a) + s) with a = 1 + 2^-30, s = -(1 + 2^-29): 0 when rounded, 2^-60 when fused
    assert out[4] == 2.0 ** -60, list(out)
    assert bad.tf_canary() == _lib.TF_ECANARY
    assert _lib.lib().tf_canary() == _lib.TF_OK  # the product build passes the same checks


@pytest.mark.gpu
def test_import_check_raises_on_a_failing_canary(cuda, monkeypatch):
    """ensure_canary (run at package import, kernels.py:559-568) turns TF_ECANARY into RuntimeError."""
    import paper_1401_0248_b200 as tfb
    from paper_1401_0248_b200 import _lib
    bad = ctypes.CDLL(UNSAFE)
    bad.tf_canary.restype = ctypes.c_int

    class Shim:
        def __getattr__(self, name):
            return getattr(_lib.lib(), name)

        tf_canary = staticmethod(bad.tf_canary)

    monkeypatch.setattr(_lib, "_canary_ok", set())
    monkeypatch.setattr(_lib, "lib", lambda: Shim())
    with pytest.raises(RuntimeError, match="strict IEEE rounding"):
        tfb._import_canary()
