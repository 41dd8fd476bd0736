# Short-row kernel variants (scripts/build_rs_variants.sh) over the row shapes; TFB_ROWS=1 = CTA-per-row kernels.
mkdir -p gpurun_out/rs
timeout 300 python scripts/rows_shapes.py > gpurun_out/rs/default.txt 2>&1
TFB_ROWS=2 timeout 300 python scripts/rows_shapes.py > gpurun_out/rs/force_short.txt 2>&1
TFB_ROWS=1 timeout 300 python scripts/rows_shapes.py 1 > gpurun_out/rs/cta_ldg.txt 2>&1
for f in paper_1401_0248_b200/variants/libtwofold_b200_rs_*.so; do
  t=$(basename $f .so)
  TFB_LIB=$PWD/$f timeout 300 python scripts/rows_shapes.py > gpurun_out/rs/$t.txt 2>&1
done
for f in gpurun_out/rs/*.txt; do echo "== $f"; awk '{print $1, $2, $4, $7, $9, substr($10,1,40)}' $f; done
