# Round-2 ncu evidence for the default bench (cfg5 as stated, 2^32): launch list of the bench
# command, one full capture of the reduction kernel (details + raw CSV), and the same for cfg2.
mkdir -p gpurun_out/r02ncu /tmp/r02ncu
C="python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu"
$C > gpurun_out/r02ncu/plain.json 2> gpurun_out/r02ncu/plain.err && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02ncu/launches_cfg5.csv $C > gpurun_out/r02ncu/launch.log 2>&1; echo launches rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:leaves -s 3 -c 1 \
  -o /tmp/r02ncu/cfg5 $C > gpurun_out/r02ncu/full.log 2>&1; echo full rc=$?
ncu -i /tmp/r02ncu/cfg5.ncu-rep --page details > gpurun_out/r02ncu/cfg5_details.txt 2>&1
ncu -i /tmp/r02ncu/cfg5.ncu-rep --page raw --csv > gpurun_out/r02ncu/cfg5_raw.csv 2>&1
C2="python bench.py --config cfg2 --steps 5 --warmup 3 --no-e2e --no-cpu"
$C2 > gpurun_out/r02ncu/plain2.json 2>/dev/null && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:leaves -s 6 -c 1 \
    -o /tmp/r02ncu/cfg2 $C2 > gpurun_out/r02ncu/full2.log 2>&1; echo full2 rc=$?
ncu -i /tmp/r02ncu/cfg2.ncu-rep --page details > gpurun_out/r02ncu/cfg2_details.txt 2>&1
ncu -i /tmp/r02ncu/cfg2.ncu-rep --page raw --csv > gpurun_out/r02ncu/cfg2_raw.csv 2>&1
ls -la gpurun_out/r02ncu
