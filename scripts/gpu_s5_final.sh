# Session-5 final check: full GPU suite (release + the device-assert build on the parity suites), smoke, ncu evidence of the default bench
# (launch list + one full capture of the TMA kernel), bench lines: reference arm, default, every config.
mkdir -p gpurun_out/s5final /tmp/s5final
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 | tee gpurun_out/s5final/gputests.txt
TFB_LIB=$PWD/paper_1401_0248_b200/csrc/build/debug/libtwofold_b200_debug.so python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_hybrid.py tests/test_gpu_dropin.py tests/test_gpu_baseline_configs.py -x -q 2>&1 | tail -2 | tee gpurun_out/s5final/debugtests.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py --impl reference > gpurun_out/s5final/bench_reference.json 2>/dev/null
python bench.py > gpurun_out/s5final/bench_default.json 2>/dev/null
for c in cfg1 cfg2 cfg2-small cfg2-dott cfg3 cfg3-sumk cfg4 cfg5-weak; do
  python bench.py --config $c --steps 50 --warmup 5 2>/dev/null >> gpurun_out/s5final/bench_configs.jsonl
done
C="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
$C > gpurun_out/s5final/plain.json 2> gpurun_out/s5final/plain.err && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/s5final/launches_cfg5.csv $C > gpurun_out/s5final/launch.log 2>&1; echo launches rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:leaves -s 3 -c 1 \
  -o /tmp/s5final/cfg5 $C > gpurun_out/s5final/full.log 2>&1; echo full rc=$?
ncu -i /tmp/s5final/cfg5.ncu-rep --page details > gpurun_out/s5final/cfg5_details.txt 2>&1
ncu -i /tmp/s5final/cfg5.ncu-rep --page raw --csv > gpurun_out/s5final/cfg5_raw.csv 2>&1
ls -la gpurun_out/s5final
