# Unroll/pipeline variant sweep at the leaf sizes that matter (results -> gpurun_out/var/)
mkdir -p gpurun_out/var
for so in paper_1401_0248_b200/variants/*.so; do
  tag=$(basename $so .so | sed 's/libtwofold_b200_//')
  for spec in "cfg2 13" "cfg2 14" "cfg2 15" "cfg2-dott 15" "cfg5 16" "cfg3 16" "cfg3-sumk 16" "cfg4 16" "cfg1 11" "cfg1 12" "cfg2-small 10"; do
    set -- $spec
    TFB_LIB=$so python bench.py --config $1 --leaf-log2 $2 --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/var/$tag.$1.$2.json 2> gpurun_out/var/$tag.$1.$2.err
  done
done
python - <<'PY'
import json, glob, os, collections
res = collections.defaultdict(dict)
for f in sorted(glob.glob("gpurun_out/var/*.json")):
    b = os.path.basename(f)[:-5]
    tag, rest = b.split(".", 1)
    try:
        d = json.load(open(f)); res[rest][tag] = 1e3 * d["roofline"]["kernel_ms"]
    except Exception as e:
        res[rest][tag] = None
tags = sorted({t for r in res.values() for t in r})
print("case".ljust(18) + "".join(t.rjust(12) for t in tags))
for k in sorted(res):
    print(k.ljust(18) + "".join(("%.2f" % res[k][t] if res[k].get(t) else "ERR").rjust(12) for t in tags))
PY
