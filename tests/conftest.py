"""Shared test configuration.

Markers: `gpu` tests need a B200 and the built CUDA library; everything else
runs on CPU (oracle vs golden fixtures, host logic, C-ABI exports, gloo
world_size-2 shard plumbing, SASS checks).
"""

import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built .so")
    config.addinivalue_line("markers", "slow: large CPU-side oracle work")
    _ensure_built()


def _ensure_built():
    """Built libraries are git-ignored: build them once if a fresh checkout lacks them
    (nvcc cross-compiles sm_100a without a GPU; the oracle is plain gcc)."""
    import subprocess
    so = os.path.join(REPO, "paper_1401_0248_b200", "libtwofold_b200.so")
    tfo = os.path.join(REPO, "oracle", "build", "libtfo.so")
    if not os.path.exists(tfo):
        subprocess.run(["make", "-s", "-C", os.path.join(REPO, "oracle")], check=True)
    if not os.path.exists(so):
        subprocess.run(["make", "-s", "-j4", "-C", os.path.join(REPO, "paper_1401_0248_b200", "csrc")], check=True)


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


@pytest.fixture(scope="session")
def golden():
    import json
    with open(os.path.join(REPO, "tests", "golden", "reference_outputs.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test selected but no CUDA device is visible")
    return torch.device("cuda", 0)
