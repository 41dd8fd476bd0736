# Hybrid host path: parity tests, then the e2e line vs host-worker count (cfg5-weak = 2^29 f64 dot).
mkdir -p gpurun_out/hybrid
timeout 900 python -m pytest tests/test_gpu_hybrid.py tests/test_host_leaves.py -q -x 2>&1 | tail -3
for t in 0 4 8 15; do
  TFB_HYBRID_THREADS=$t timeout 600 python bench.py --config cfg5-weak --steps 10 --warmup 3 --no-cpu \
    > gpurun_out/hybrid/e2e_t$t.json 2> gpurun_out/hybrid/e2e_t$t.err
  python -c "import json; d=json.load(open('gpurun_out/hybrid/e2e_t$t.json')); e=d['e2e']; print('threads $t', round(e['value'],3), 'Gelem/s host_share', round(e.get('host_share',0),3), 'h2d/step', e['h2d_bytes_per_step'], 'ms', round(e['ms_per_step'],1))" 2>&1 | tail -1
done
