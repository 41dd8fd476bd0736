set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo rc=$?
for c in cfg1 cfg2 cfg2-dott cfg2-small cfg3 cfg3-sumk cfg4; do
  python bench.py --config $c --steps 50 --warmup 5 --no-cpu --no-e2e > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c rc=$?
done
tail -c 3000 gpurun_out/bench_cfg5.err
