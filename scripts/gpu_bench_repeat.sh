# The default bench line five times in a row (run-to-run spread of the headline number).
mkdir -p gpurun_out/repeat
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/repeat/run$i.json 2>/dev/null
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob("gpurun_out/repeat/run*.json")):
    d = json.load(open(f)); r = d["roofline"]
    print(f.split("/")[-1], round(d["value"], 1), "Gelem/s", round(r["achieved"]), "GB/s kernel",
          round(r["frac_of_read_roof"], 4), "of read roof", d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
