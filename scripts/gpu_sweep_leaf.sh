# Leaf-size sweep for the small/medium configs (methodology: rotation + CUDA graph).
mkdir -p gpurun_out/sweep
for c in cfg1 cfg2 cfg2-small cfg2-dott; do
  for lg in 0 10 11 12 13 14 15 16; do
    python bench.py --config $c --steps 50 --warmup 3 --no-cpu --no-e2e --leaf-log2 $lg > gpurun_out/sweep/$c.$lg.json 2> gpurun_out/sweep/$c.$lg.err
  done
done
for c in cfg3 cfg4 cfg5; do
  for lg in 0 14 15 16 17 18; do
    python bench.py --config $c --steps 30 --warmup 3 --no-cpu --no-e2e --leaf-log2 $lg > gpurun_out/sweep/$c.$lg.json 2> gpurun_out/sweep/$c.$lg.err
  done
done
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob("gpurun_out/sweep/*.json")):
    try:
        d = json.load(open(f))
        r = d["roofline"]
        print(os.path.basename(f), "leaf", d["config"]["leaf_log2"], "kernel_us %.2f" % (1e3 * r["kernel_ms"]), "GB/s %.0f" % r["achieved"], "frac %.3f" % r["frac"])
    except Exception as e:
        print(os.path.basename(f), "ERR", e, open(f.replace(".json", ".err")).read()[-300:])
PY
