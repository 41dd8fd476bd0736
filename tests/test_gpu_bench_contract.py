"""bench.py keeps the driver's JSON-line contract (one line on stdout, every key the
contract names, sane values) — on a quick config, ours and the reference arm."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                         timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout[-2000:]  # exactly one JSON line on stdout
    return json.loads(lines[0])


def test_bench_line_contract(cuda):
    d = _run("--config", "cfg2-small", "--steps", "5", "--warmup", "3")
    assert KEYS <= set(d), KEYS - set(d)
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["unit"] == "Gelem/s" and d["dtype"] == "f32"
    assert d["scaling"] in ("weak", "strong") and d["data"] == "synthetic" and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["unit"] == "GB/s" and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-6
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == 2 * 4 * (1 << 16) and e["d2h_bytes_per_step"] == 16
    c = d["cpu_baseline"]
    assert c["value"] > 0 and c["cores"] >= 1 and c["kind"] in ("port", "reference") and c["sample"]
    assert d["gpu_launches"] >= d["steps"]  # our kernels, counted inside the timed region
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


def test_reference_arm_contract(cuda):
    d = _run("--impl", "reference", "--config", "cfg2-small", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "Gelem/s"
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["kind"] in ("port", "reference")


def test_self_launch_through_torchrun_with_the_collective(cuda):
    """--gpus 1 --spawn re-executes under torch.distributed.run; --force-collective runs the
    NCCL all-gather + merge kernel in every step at world size 1 (the N>1 code path)."""
    d = _run("--gpus", "1", "--spawn", "--force-collective", "--config", "cfg5-weak", "--steps", "3", "--warmup", "3",
             "--no-cpu", "--no-e2e")
    assert d["n_gpus"] == 1 and d["value"] > 100 and "NCCL" in d["run"]["combine"]
    assert d["roofline"]["kernel_ms"] <= d["ms_per_step"] * 1.001
    assert d["config"]["n_per_rank"] == 1 << 29 and d["scaling"] == "weak"
