mkdir -p gpurun_out/ncu2
python scripts/exact_one.py > gpurun_out/ncu2/exact_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none -k regex:exact_kernel -s 2 -c 1 -o gpurun_out/ncu2/prof_exact python scripts/exact_one.py > gpurun_out/ncu2/exact_ncu.log 2>&1; echo exact rc=$?
if [ -f gpurun_out/ncu2/prof_exact.ncu-rep ]; then
  ncu -i gpurun_out/ncu2/prof_exact.ncu-rep --page raw --csv > gpurun_out/ncu2/prof_exact_raw.csv 2>/dev/null
  ncu -i gpurun_out/ncu2/prof_exact.ncu-rep --page details > gpurun_out/ncu2/prof_exact_details.txt 2>/dev/null
  rm -f gpurun_out/ncu2/prof_exact.ncu-rep
fi
