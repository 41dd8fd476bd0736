# Session-5 ncu evidence: cfg2 after the L2 prefetch preamble / re-tuned loader table (launch list of the bench command,
# one full capture of the leaves kernel), plus bench lines for every BASELINE config.
mkdir -p gpurun_out/s5ncu /tmp/s5ncu
C2="python bench.py --config cfg2 --steps 5 --warmup 3 --no-e2e --no-cpu"
$C2 > gpurun_out/s5ncu/plain2.json 2>/dev/null && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/s5ncu/launches_cfg2.csv $C2 > gpurun_out/s5ncu/launch2.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaves_kernel -s 6 -c 1 \
    -o /tmp/s5ncu/cfg2 $C2 > gpurun_out/s5ncu/full2.log 2>&1; echo full2 rc=$?
ncu -i /tmp/s5ncu/cfg2.ncu-rep --page details > gpurun_out/s5ncu/cfg2_details.txt 2>&1
ncu -i /tmp/s5ncu/cfg2.ncu-rep --page raw --csv > gpurun_out/s5ncu/cfg2_raw.csv 2>&1
for c in cfg1 cfg2 cfg2-small cfg2-dott cfg3 cfg3-sumk cfg4; do
  python bench.py --config $c --steps 50 --warmup 5 2>/dev/null >> gpurun_out/s5ncu/bench_configs.jsonl
done
python bench.py --impl reference > gpurun_out/s5ncu/bench_reference.json 2>/dev/null
python bench.py > gpurun_out/s5ncu/bench_default.json 2>/dev/null
ls -la gpurun_out/s5ncu
