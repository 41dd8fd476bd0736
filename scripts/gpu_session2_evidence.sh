# Session-2 evidence: every BASELINE config's bench line, ncu captures of the new kernels
# (lane-group rows, sequential ring), debug-build sanitize workload.
mkdir -p gpurun_out/s2
python bench.py --steps 50 --warmup 5 > gpurun_out/s2/bench_cfg5.json 2> gpurun_out/s2/bench_cfg5.err; echo cfg5 rc=$?
for c in cfg1 cfg2 cfg2-dott cfg2-small cfg3 cfg3-sumk cfg4; do
  python bench.py --config $c --steps 50 --warmup 5 > gpurun_out/s2/bench_$c.json 2> gpurun_out/s2/bench_$c.err; echo $c rc=$?
done
python scripts/rows_one.py 1048576 256 > gpurun_out/s2/rows_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:rows_short -s 2 -c 1 \
    -o gpurun_out/s2/prof_rows_short python scripts/rows_one.py 1048576 256 > gpurun_out/s2/rows_ncu.log 2>&1; echo rows ncu rc=$?
python scripts/seq_speed.py > gpurun_out/s2/seq_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none -k regex:seq_pipe -s 1 -c 1 \
    -o gpurun_out/s2/prof_seq_pipe python scripts/seq_speed.py > gpurun_out/s2/seq_ncu.log 2>&1; echo seq ncu rc=$?
# keep gpurun_out small (<= 64 MiB merge limit): text exports only
for r in prof_rows_short prof_seq_pipe; do
  if [ -f gpurun_out/s2/$r.ncu-rep ]; then
    ncu -i gpurun_out/s2/$r.ncu-rep --page raw --csv > gpurun_out/s2/${r}_raw.csv 2>/dev/null
    ncu -i gpurun_out/s2/$r.ncu-rep --page details > gpurun_out/s2/${r}_details.txt 2>/dev/null
    rm -f gpurun_out/s2/$r.ncu-rep
  fi
done
if [ -f paper_1401_0248_b200/variants/libtwofold_b200_debug.so ]; then
  TFB_LIB=$PWD/paper_1401_0248_b200/variants/libtwofold_b200_debug.so timeout 600 python scripts/sanitize_workload.py 2>&1 | tail -2
fi
