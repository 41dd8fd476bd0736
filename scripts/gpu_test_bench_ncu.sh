# Round check: GPU tests, default bench line, then ncu evidence (launch list + full capture).
mkdir -p gpurun_out/ncu
python -m pytest tests -m gpu -q 2>&1 | tail -4
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
C5="python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu"
C2="python bench.py --config cfg2 --steps 5 --warmup 2 --no-e2e --no-cpu"
$C5 > gpurun_out/ncu/plain5.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/launches_cfg5.csv $C5 > gpurun_out/ncu/launch5.log 2>&1; echo launches rc=$?
$C5 > gpurun_out/ncu/plain5b.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:leaves_kernel -s 2 -c 1 -o gpurun_out/ncu/prof_cfg5 $C5 > gpurun_out/ncu/full5.log 2>&1; echo full5 rc=$?
$C2 > gpurun_out/ncu/plain2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:leaves_kernel -s 4 -c 1 -o gpurun_out/ncu/prof_cfg2 $C2 > gpurun_out/ncu/full2.log 2>&1; echo full2 rc=$?
ls -la gpurun_out/ncu
