# LDG vs TMA-pipeline loaders (bit-identical) on every config; then the GPU tests.
mkdir -p gpurun_out/loader
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for ld in 0 1 2 3; do
  for c in cfg1 cfg2-small cfg2 cfg2-dott cfg3 cfg3-sumk cfg4 cfg5; do
    TFB_LOADER=$ld timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/loader/$c.$ld.json 2> gpurun_out/loader/$c.$ld.err
  done
done
python - <<'PY'
import json, glob, os, collections
res = collections.defaultdict(dict)
for f in glob.glob("gpurun_out/loader/*.json"):
    c, ld = os.path.basename(f)[:-5].rsplit(".", 1)
    try:
        d = json.load(open(f)); res[c][ld] = (1e3 * d["roofline"]["kernel_ms"], d["roofline"]["achieved"])
    except Exception: res[c][ld] = None
print("config".ljust(12) + "".join(f"loader={s} (us, GB/s)".rjust(26) for s in "012"))
for c in sorted(res):
    print(c.ljust(12) + "".join((("%.2f / %.0f" % res[c][s]) if res[c].get(s) else "ERR").rjust(26) for s in "012"))
PY
