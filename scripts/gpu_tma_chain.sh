python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py tests/test_gpu_fuzz.py -x -q -k "tma or cfg4 or cfg5 or rerun or fuzz" 2>&1 | tail -2
for tc in 0 1 0 1; do
  echo "== TFB_TMA_CHAIN=$tc"
  TFB_TMA_CHAIN=$tc python scripts/prefetch_sweep.py --loaders 2 --kb -1 --lo 26 --hi 31 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: r=json.loads(l)
    except Exception: continue
    print(r['dtype'],'dot' if r['dot'] else 'sum','2^%d B'%r['bytes_log2'],' '.join('%s=%.2f'%(k,v) for k,v in r['us'].items()))
" | grep dot
  for c in cfg4 cfg5-weak; do TFB_TMA_CHAIN=$tc python bench.py --config $c --steps 50 --warmup 5 --no-e2e --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('tma_chain=$tc', d['config']['workload'][:10], round(d['ms_per_step']*1e3,2), 'us', round(d['roofline']['achieved']), 'GB/s')"; done
done
