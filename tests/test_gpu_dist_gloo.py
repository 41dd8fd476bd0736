"""The shard layer (dist.sharded_reduce / sharded_rows / sharded_run) with REAL kernels at world
sizes 2 and 3 on the single test GPU: torchrun ranks that all use cuda:0 over a gloo process group
(scripts/dist_gloo_gpu_check.py).  The CPU twin of this test (tests/test_dist_gloo.py) replaces the
kernels by their oracle restatements; here nothing is replaced."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world", [2, 3])
def test_shard_layer_real_kernels_world_gt_1(cuda, world):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29570 + world),
           os.path.join(REPO, "scripts", "dist_gloo_gpu_check.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=REPO)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert f"gloo shard layer ok" in out.stdout and f"world {world}" in out.stdout
