"""Register budgets of the streaming kernels (occupancy is the LDG loader's
bytes-in-flight): a regression here silently costs a CTA per SM (this happened
once — an inlined cross-GPU path took leaves_kernel from 48 to 62 registers)."""

import os
import re
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(REPO, "paper_1401_0248_b200", "libtwofold_b200.so")


@pytest.fixture(scope="module")
def regs():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not installed")
    out = subprocess.run(["cuobjdump", "-res-usage", SO], capture_output=True, text=True, check=True).stdout
    res, fn = {}, None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            fn = m.group(1)
            continue
        m = re.search(r"REG:(\d+)", line)
        if m and fn:
            res[fn] = int(m.group(1))
    return res


def test_ldg_leaves_kernels_keep_five_ctas_per_sm(regs):
    # leaves_kernel<M, T, DOT, VEC=1, NT=256>: <= 51 registers -> 5 CTAs x 256 threads per SM
    vec256 = {f: r for f, r in regs.items() if re.search(r"leaves_kernelILi[0-6]E[fd]Lb[01]ELb1ELi256ELi1E", f)}
    assert len(vec256) >= 19
    over = {f: r for f, r in vec256.items() if r > 51}
    # the rigorous/TwoProduct f64 dots are allowed up to 64 (4 CTAs/SM); everything else 5
    over = {f: r for f, r in over.items() if not (re.search(r"ILi[36]EdLb1E", f) and r <= 64)}
    assert not over, over


def test_tma_kernels_fit_one_cta_per_sm(regs):
    tma = {f: r for f, r in regs.items() if "leaves_tma_kernel" in f}
    assert tma and max(tma.values()) <= 224  # 288 threads x 224 <= 65536


def test_deep_ldg_variants_keep_four_ctas_per_sm(regs):
    # leaves_kernel<..., NT=256, UF=2>: twice the loads in flight, <= 64 registers (4 CTAs/SM)
    deep = {f: r for f, r in regs.items() if re.search(r"leaves_kernelILi[0-6]E[fd]Lb[01]ELb1ELi256ELi2E", f)}
    assert len(deep) >= 19
    assert max(deep.values()) <= 64, {f: r for f, r in deep.items() if r > 64}
