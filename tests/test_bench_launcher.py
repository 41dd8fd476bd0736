"""bench.py's launcher on CPU: `--gpus N` without a torchrun environment re-executes itself
under torch.distributed.run with N ranks; --dry-run joins a gloo group on every rank and
rank 0 prints ONE JSON line whose n_gpus is the world size (no GPU work)."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "TFB_BENCH_CHILD")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                         timeout=300, cwd=REPO, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_gpus_2_self_launches_two_ranks():
    d = _run("--gpus", "2", "--dry-run", "--steps", "1", "--warmup", "0")
    assert d["n_gpus"] == 2 and d["dry_run"] is True and d["rank_sum"] == 1  # ranks 0 + 1 joined
    assert d["config"]["n_global"] == 1 << 32 and d["config"]["n_per_rank"] == 1 << 31  # cfg5 as stated, split
    assert d["scaling"] == "strong" and "dp2" in d["config"]["parallelism"]


def test_spawn_at_one_gpu_uses_the_same_path():
    d = _run("--gpus", "1", "--spawn", "--dry-run", "--steps", "1", "--warmup", "0")
    assert d["n_gpus"] == 1 and d["config"]["n_per_rank"] == 1 << 32


def test_weak_workload_and_identical_config_between_arms():
    """Both arms describe the workload with the SAME config dict (same_config)."""
    sys.path.insert(0, REPO)
    import bench
    from paper_1401_0248_b200.gen import CONFIGS
    for world in (1, 2, 8):
        a = bench.workload_desc("cfg5", CONFIGS["cfg5"], "twofold-fast", world)
        assert a["n_global"] == 1 << 32 and a["n_per_rank"] == (1 << 32) // world
        w = bench.workload_desc("cfg5-weak", CONFIGS["cfg5"], "twofold-fast", world)
        assert w["n_per_rank"] == 1 << 29 and w["n_global"] == (1 << 29) * world
    d = _run("--gpus", "1", "--dry-run", "--config", "cfg5-weak", "--steps", "1", "--warmup", "0")
    assert d["scaling"] == "weak" and d["config"] == bench.workload_desc("cfg5-weak", CONFIGS["cfg5"],
                                                                          "twofold-fast", 1)
