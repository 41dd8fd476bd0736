# Default bench (cfg5 as stated, 2^32 on one GPU), the reference arm, and the hybrid at 15/16 host workers.
mkdir -p gpurun_out/r02b
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02b/bench_default.json 2> gpurun_out/r02b/bench_default.err; echo bench rc=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02b/bench_reference.json 2> gpurun_out/r02b/bench_reference.err; echo ref rc=$?
TFB_HYBRID_THREADS=16 timeout 600 python bench.py --config cfg5-weak --steps 10 --warmup 3 --no-cpu > gpurun_out/r02b/e2e_t16.json 2>/dev/null; echo t16 rc=$?
python - <<'PY'
import json
for f in ("bench_default", "bench_reference", "e2e_t16"):
    d = json.load(open(f"gpurun_out/r02b/{f}.json"))
    r = d.get("roofline") or {}
    e = d.get("e2e") or {}
    print(f, "value", round(d["value"], 2), "ms/step", round(d["ms_per_step"], 3), "kernel_ms", r.get("kernel_ms"),
          "frac", r.get("frac"), "read-roof frac", r.get("frac_of_read_roof"), "e2e", e.get("value"),
          "host_share", e.get("host_share"), "cpu", (d.get("cpu_baseline") or {}).get("value"), d.get("clocks"))
PY
