# Round-2 check: GPU tests, smoke, default bench (cfg5 as stated, 2^32 on one GPU),
# the reference arm, the self-launch path, host facts.
mkdir -p gpurun_out/r02
{ free -g; nproc; lscpu | grep -E "Model name|Socket|NUMA|Thread"; cat /sys/kernel/mm/transparent_hugepage/enabled; } > gpurun_out/r02/host.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02/bench_default.json 2> gpurun_out/r02/bench_default.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02/bench_reference.json 2> gpurun_out/r02/bench_reference.err; echo ref rc=$?
timeout 600 python bench.py --gpus 1 --spawn --config cfg5-weak --steps 20 --warmup 5 --force-collective --no-cpu > gpurun_out/r02/bench_spawn.json 2> gpurun_out/r02/bench_spawn.err; echo spawn rc=$?
python - <<'PY'
import json
for f in ("bench_default", "bench_reference", "bench_spawn"):
    try:
        d = json.load(open(f"gpurun_out/r02/{f}.json"))
    except Exception as e:
        print(f, "unreadable", e); continue
    r = d.get("roofline") or {}
    print(f, "value", round(d["value"], 2), "n_gpus", d["n_gpus"], "ms/step", round(d["ms_per_step"], 3),
          "kernel_ms", r.get("kernel_ms"), "frac", r.get("frac"), "read roof frac", r.get("frac_of_read_roof"),
          "e2e", (d.get("e2e") or {}).get("value"), "cpu", (d.get("cpu_baseline") or {}).get("value"),
          "1core", ((d.get("cpu_baseline") or {}).get("single_core") or {}).get("value"), d.get("clocks"))
PY
