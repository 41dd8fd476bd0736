# A/B of the loaders on cfg3 (sumt, sumk) through bench.py, 3 repeats each, alternating.
mkdir -p gpurun_out/ab
for rep in 1 2 3; do
  for ld in 1 2; do
    for c in cfg3 cfg3-sumk; do
      TFB_LOADER=$ld timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/ab/$c.$ld.$rep.json 2>/dev/null
    done
  done
done
python - <<'PY'
import json, glob, os, collections
res = collections.defaultdict(list)
for f in glob.glob("gpurun_out/ab/*.json"):
    c, ld, rep = os.path.basename(f)[:-5].split(".")
    d = json.load(open(f)); res[(c, ld)].append(1e3 * d["roofline"]["kernel_ms"])
for k in sorted(res): print(k, ["%.1f" % v for v in sorted(res[k])])
PY
