"""Fused NVLink peer combine (tf_reduce_peer) on the GPU through torchrun + NCCL
process groups: bit-identical to the NCCL all-gather path (world size 1 on the
single-GPU test box; the same script runs at any --nproc-per-node)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_peer_combine_matches_nccl(cuda):
    import torch
    n = torch.cuda.device_count()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={min(n, 8)}",
           "--master-addr", "127.0.0.1", "--master-port", "29561", os.path.join(REPO, "scripts", "peer_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "peer combine ok" in out.stdout
