"""The C ABI from native code: examples/reduce_example.c compiles against
include/twofold_b200.h + the in-tree .so (CPU), and runs on a B200 (gpu)."""

import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = "/usr/local/cuda"


def _build(tmp_path):
    cc = shutil.which("gcc") or shutil.which("cc")
    if not cc or not os.path.isdir(os.path.join(CUDA, "include")):
        pytest.skip("no C compiler or CUDA headers")
    exe = str(tmp_path / "reduce_example")
    lib = os.path.join(REPO, "paper_1401_0248_b200")
    cmd = [cc, "-O2", os.path.join(REPO, "examples", "reduce_example.c"), "-I", os.path.join(REPO, "include"),
           "-I", f"{CUDA}/include", "-L", lib, "-ltwofold_b200", "-L", f"{CUDA}/lib64", "-lcudart",
           f"-Wl,-rpath,{lib}:{CUDA}/lib64", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_native_example_builds(tmp_path):
    assert os.path.exists(_build(tmp_path))


@pytest.mark.gpu
def test_native_example_runs(tmp_path, cuda):
    exe = _build(tmp_path)
    out = subprocess.run([exe, str(1 << 22)], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "value=" in out.stdout and "leaves_" in out.stdout and "bit-identical" in out.stdout
