# Round check: GPU tests, default bench line, ncu launch list + full capture of the top kernel.
mkdir -p gpurun_out/ncu
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
C5="python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu"
$C5 > gpurun_out/ncu/plain5.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_cfg5.csv $C5 > gpurun_out/ncu/launch5.log 2>&1; echo launches rc=$?
$C5 > gpurun_out/ncu/plain5b.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaves -s 2 -c 1 -o gpurun_out/ncu/prof_cfg5_tma $C5 > gpurun_out/ncu/full5.log 2>&1; echo full5 rc=$?
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_default.json"))
print({k: d[k] for k in ("value", "ms_per_step", "hbm_gbs")}, d["roofline"]["achieved"], d["roofline"]["frac"], d["e2e"]["value"], d["cpu_baseline"]["value"], d["clocks"])
PY
