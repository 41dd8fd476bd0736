# GPU tests + one bench line per config (kernel µs), results in gpurun_out/quick/
mkdir -p gpurun_out/quick
python -m pytest tests -m gpu -q 2>&1 | tail -4
for c in cfg1 cfg2-small cfg2 cfg2-dott cfg3 cfg3-sumk cfg4 cfg5; do
  python bench.py --config $c --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/quick/$c.json 2> gpurun_out/quick/$c.err
done
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob("gpurun_out/quick/*.json")):
    try:
        d = json.load(open(f)); r = d["roofline"]
        print(os.path.basename(f)[:-5].ljust(12), "kernel %.2f us" % (1e3 * r["kernel_ms"]), "%.0f GB/s" % r["achieved"], "frac %.3f" % r["frac"], "value %.1f Gelem/s" % d["value"])
    except Exception as e:
        print(f, "ERR", open(f.replace(".json", ".err")).read()[-400:])
PY
