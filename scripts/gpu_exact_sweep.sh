for f in paper_1401_0248_b200/variants/libtwofold_b200_ex_*.so; do
  echo "== $(basename $f .so)"
  TFB_LIB=$PWD/$f timeout 300 python scripts/exact_bench.py 2>&1 | awk '{print $1, $2, $3, $5, $6}'
done
