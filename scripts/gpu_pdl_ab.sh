# A/B of the cross-call PDL chain (TFB_PDL_CHAIN) on the graph-replayed small/mid configs, interleaved.
for rep in 1 2 3; do
  for c in cfg2 cfg2-dott cfg1 cfg2-small; do
    for v in 0 1; do
      TFB_PDL_CHAIN=$v timeout 300 python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e 2>/dev/null | \
        python -c "import json,sys; d=json.load(sys.stdin); print('$c chain=$v', round(d['ms_per_step']*1e3,2), 'us')"
    done
  done
done
