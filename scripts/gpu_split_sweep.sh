# Leaf-split sweep (result-neutral grid balancing), then the GPU tests.
mkdir -p gpurun_out/split
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for sp in 0 1 2 4; do
  for c in cfg1 cfg2-small cfg2 cfg2-dott cfg3 cfg4 cfg5; do
    TFB_SPLIT=$sp python bench.py --config $c --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/split/$c.$sp.json 2> gpurun_out/split/$c.$sp.err
  done
done
python - <<'PY'
import json, glob, os, collections
res = collections.defaultdict(dict)
for f in glob.glob("gpurun_out/split/*.json"):
    c, sp = os.path.basename(f)[:-5].rsplit(".", 1)
    try: res[c][sp] = 1e3 * json.load(open(f))["roofline"]["kernel_ms"]
    except Exception as e: res[c][sp] = None
print("config".ljust(12) + "".join(f"split={s}".rjust(12) for s in "0124"))
for c in sorted(res):
    print(c.ljust(12) + "".join((("%.2f" % res[c][s]) if res[c].get(s) else "ERR").rjust(12) for s in "0124"))
PY
