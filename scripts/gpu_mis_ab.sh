# Misaligned-rows A/B over library variants (TFB_LIB), rows_mis_ab.py each.
for lib in "" $(ls paper_1401_0248_b200/csrc/build/variants/*.so 2>/dev/null); do
  echo "== lib ${lib:-default}"
  env ${lib:+TFB_LIB=$PWD/$lib} python scripts/rows_mis_ab.py 2>&1
done
