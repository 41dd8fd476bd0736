# A/B of the cross-call PDL chain on the large eager-timed configs, interleaved.
for rep in 1 2; do
  for c in cfg3 cfg3-sumk cfg4 cfg5-weak; do
    for v in 0 1; do
      TFB_PDL_CHAIN=$v timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu --no-e2e 2>/dev/null | \
        python -c "import json,sys; d=json.load(sys.stdin); print('$c chain=$v', round(d['ms_per_step']*1e3,2), 'us', d['roofline']['kernel'][:60])"
    done
  done
done
