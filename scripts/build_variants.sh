# Build tuning variants of the library (unroll depth x software pipeline) into
# paper_1401_0248_b200/variants/, selected at run time with TFB_LIB=<path>.
set -e
cd "$(dirname "$0")/../paper_1401_0248_b200/csrc"
mkdir -p ../variants
for v in "4 2 1" "2 1 1" "8 4 1" "2 2 1" "4 4 0" "8 4 0" "4 2 0"; do
  set -- $v
  tag="u$1_$2_p$3"
  rm -rf build_$tag; mkdir -p build_$tag
  for f in reduce misc exact host; do
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
      -lineinfo -Xcompiler -fPIC -I../../include -DTFB_UNROLL_F32=$1 -DTFB_UNROLL_F64=$2 -DTFB_PIPELINE=$3 \
      -c $f.cu -o build_$tag/$f.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../variants/libtwofold_b200_$tag.so build_$tag/*.o
  rm -rf build_$tag
done
ls ../variants
