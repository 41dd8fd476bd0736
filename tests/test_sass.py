"""Codegen guard (the device analogue of the fast-math canary, kernels.py:545-568).

Every reduction kernel must be built from separate IEEE adds/multiplies: a
contracted FFMA/DFMA in a reduction path would change the dot products'
rounding (the reference rounds each product, kernels.py:23-26) and an
FTZ/fast-math build would zero the error channel.  The hot kernels must use
the 128-bit streaming load path.
"""

import os
import re
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(REPO, "paper_1401_0248_b200", "libtwofold_b200.so")


@pytest.fixture(scope="module")
def sass():
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not installed")
    out = subprocess.run(["cuobjdump", "-sass", SO], check=True, capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in out.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    return funcs


REDUCTION = ("leaves_kernel", "leaves_tma_kernel", "small_cluster_kernel", "tree_kernel", "rows_tree_kernel", "seq_kernel",
             "lanes_kernel",
             "canary_kernel", "eft_kernel", "noread_kernel")


def test_sm100a_code_present(sass):
    assert any("leaves_kernel" in f for f in sass)
    arch = subprocess.run(["cuobjdump", "-lelf", SO], capture_output=True, text=True).stdout
    assert "sm_100a" in arch


def _is_two_product(fn):
    # internal method ids 5/6 (kFastTP / kRigorousTP) are the opt-in TwoProduct dots
    return bool(re.search(r"kernelILi[56]E", fn))


def test_two_product_kernels_use_fma(sass):
    # kernels that accumulate elements (the tree kernels only merge pairs)
    tp = [fn for fn in sass if _is_two_product(fn) and "tree_kernel" not in fn]
    assert len(tp) >= 12
    for fn in tp:
        assert any(re.search(r"\b(DFMA|FFMA)\b", ln) for ln in sass[fn]), fn


def test_no_fused_multiply_add_in_reduction_kernels(sass):
    bad = []
    for fn, lines in sass.items():
        if any(k in fn for k in REDUCTION) and not _is_two_product(fn):
            for ln in lines:
                if re.search(r"\b(FFMA|DFMA|FFMA2)\b", ln):
                    bad.append((fn, ln.strip()))
                # HFMA2 Rd, -RZ, RZ, imm is ptxas's register-move idiom, not arithmetic
                elif re.search(r"\bHFMA2\b", ln) and "-RZ, RZ" not in ln:
                    bad.append((fn, ln.strip()))
    assert not bad, bad[:5]


def test_no_flush_to_zero_arithmetic(sass):
    for fn, lines in sass.items():
        if any(k in fn for k in REDUCTION):
            # floating-point arithmetic must keep subnormals (F2I.FTZ of the integer
            # division idiom is a conversion, not data arithmetic)
            assert not any(re.search(r"\b(FADD|FMUL|DADD|DMUL|FSETP|FMNMX)\S*\.FTZ", ln) for ln in lines), fn


def test_streaming_128bit_loads_in_vector_kernels(sass):
    # leaves_kernel<M, T, DOT, VEC=true, NT>
    vec = [fn for fn in sass if re.search(r"leaves_kernelILi\dE[fd]Lb[01]ELb1ELi\d+E", fn)]
    assert vec
    for fn in vec:
        assert any(re.search(r"LDG\.E\.(NA\.)?\S*128", ln) for ln in sass[fn]), fn
