# Tuning builds of the short-row kernel (rows.cuh): min CTAs/SM x load batches,
# into paper_1401_0248_b200/variants/ (select with TFB_LIB=<path>).
set -e
cd "$(dirname "$0")/../paper_1401_0248_b200/csrc"
mkdir -p ../variants
for v in "0 0" "2 0"; do
  set -- $v
  tag="rs_m$1_p$2"
  rm -rf build_$tag; mkdir -p build_$tag
  for f in reduce misc exact host; do
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
      -Xcompiler -fPIC -I../../include -DTFB_RS_MINB=$1 -DTFB_RS_PARTS=$2 -c $f.cu -o build_$tag/$f.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../variants/libtwofold_b200_$tag.so build_$tag/*.o -lpthread
  rm -rf build_$tag
done
ls ../variants
