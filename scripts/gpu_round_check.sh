# Round check: GPU tests, smoke, default bench line, reference arm, ncu launch list + full capture.
mkdir -p gpurun_out/ncu gpurun_out/final
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err; echo bench rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_reference.json 2> gpurun_out/final/bench_reference.err; echo ref rc=$?
C5="python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu"
$C5 > gpurun_out/ncu/plain5.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_cfg5.csv $C5 > gpurun_out/ncu/launch5.log 2>&1; echo launches rc=$?
$C5 > gpurun_out/ncu/plain5b.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaves -s 2 -c 1 -o gpurun_out/final/prof_cfg5 $C5 > gpurun_out/ncu/full5.log 2>&1; echo full5 rc=$?
python - <<'PY'
import json
d = json.load(open("gpurun_out/final/bench_default.json"))
r = d["roofline"]
print("ours", round(d["value"], 1), "Gelem/s", round(r["achieved"]), "GB/s frac", round(r["frac"], 3), "of read roof", r.get("frac_of_read_roof"), "e2e", round(d["e2e"]["value"], 2), "cpu", round(d["cpu_baseline"]["value"], 2), d["clocks"])
d = json.load(open("gpurun_out/final/bench_reference.json"))
print("reference arm", round(d["value"], 2), d["cpu_baseline"]["cores"])
PY
