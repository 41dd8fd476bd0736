for v in default ld_nohint ld_128b ld_evfirst; do
  if [ $v = default ]; then L=""; else L="TFB_LIB=$PWD/paper_1401_0248_b200/variants/libtwofold_b200_$v.so"; fi
  echo "== $v"
  env $L timeout 300 python scripts/latency_breakdown.py 2>&1 | grep -o "^[^|]*|[^|]*|[^|]*| PDL [0-9.]*\|auto [0-9.]*" | tr '\n' ' '; echo
  for c in cfg3 cfg2-dott; do env $L timeout 300 python bench.py --config $c --steps 20 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$c', round(d['roofline']['kernel_ms']*1e3,2), 'us')"; done
done
