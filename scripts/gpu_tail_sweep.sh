# Tail variants (last-CTA ticket vs PDL tree kernel) x leaf split, small/mid configs; then the tail test.
mkdir -p gpurun_out/tail
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "pdl or tma or split" 2>&1 | tail -3
for tl in 1 2; do
  for sp in 1 2; do
    for c in cfg1 cfg2-small cfg2 cfg3 cfg5; do
      TFB_TAIL=$tl TFB_SPLIT=$sp TFB_LOADER=1 timeout 300 python bench.py --config $c --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/tail/$c.$tl.$sp.json 2> gpurun_out/tail/$c.$tl.$sp.err
    done
  done
done
python - <<'PY'
import json, glob, os, collections
res = collections.defaultdict(dict)
for f in glob.glob("gpurun_out/tail/*.json"):
    c, tl, sp = os.path.basename(f)[:-5].rsplit(".", 2)
    try: res[c][f"t{tl}s{sp}"] = 1e3 * json.load(open(f))["roofline"]["kernel_ms"]
    except Exception: res[c][f"t{tl}s{sp}"] = None
keys = ["t1s1", "t1s2", "t2s1", "t2s2"]
print("config".ljust(12) + "".join(k.rjust(10) for k in keys))
for c in sorted(res):
    print(c.ljust(12) + "".join((("%.2f" % res[c][k]) if res[c].get(k) else "ERR").rjust(10) for k in keys))
PY
