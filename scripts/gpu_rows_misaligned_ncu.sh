# ncu of the short-rows kernel on misaligned pitches (f32 255 / 777 cols) vs aligned (256);
# the reports are summarised on the box (details + raw CSV) and the .ncu-rep files dropped.
mkdir -p gpurun_out/rowsmis /tmp/rowsmis
for shape in "262144 255" "100003 777" "262144 256" "131072 255 f64"; do
  set -- $shape
  tag="$1x$2${3:-}"
  python scripts/rows_one.py $shape > gpurun_out/rowsmis/plain_$tag.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:rows_short -s 2 -c 1 \
     -o /tmp/rowsmis/prof_$tag python scripts/rows_one.py $shape > gpurun_out/rowsmis/ncu_$tag.log 2>&1
  echo "$tag rc=$?"
  ncu -i /tmp/rowsmis/prof_$tag.ncu-rep --page details > gpurun_out/rowsmis/details_$tag.txt 2>&1
  ncu -i /tmp/rowsmis/prof_$tag.ncu-rep --page raw --csv > gpurun_out/rowsmis/raw_$tag.csv 2>&1
  ncu -i /tmp/rowsmis/prof_$tag.ncu-rep --page source --csv > gpurun_out/rowsmis/source_$tag.csv 2>&1
done
python scripts/rows_shapes.py 0 262144x255 100003x777 131072x513 1048576x63 4194304x17 > gpurun_out/rowsmis/shapes_before.txt 2>&1
du -sh gpurun_out/rowsmis
