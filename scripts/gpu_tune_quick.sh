# Re-measure the loader table (scripts/tune_loaders.py -> gpurun_out/tune/) and one bench line per big config.
mkdir -p gpurun_out/tune gpurun_out/quick
timeout 2400 python scripts/tune_loaders.py gpurun_out/tune > gpurun_out/tune/log.txt 2>&1; echo tune rc=$?
for c in cfg5 cfg3 cfg3-sumk cfg4 cfg2; do
  timeout 600 python bench.py --config $c --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/quick/$c.json 2> gpurun_out/quick/$c.err
done
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob("gpurun_out/quick/*.json")):
    try:
        d = json.load(open(f)); r = d["roofline"]
        print(os.path.basename(f)[:-5].ljust(12), "kernel %.2f us" % (1e3 * r["kernel_ms"]), "%.0f GB/s" % r["achieved"], "frac %.3f" % r["frac"], "value %.1f Gelem/s" % d["value"], r["kernel"][:60])
    except Exception as e:
        print(f, "ERR", open(f.replace(".json", ".err")).read()[-400:])
PY
