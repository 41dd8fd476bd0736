# Tuning builds of the GPU exact oracle (exact.cu): components K x load depth U x CTAs/SM.
set -e
cd "$(dirname "$0")/../paper_1401_0248_b200/csrc"
mkdir -p ../variants
for v in "4 2 4" "4 4 4" "4 1 4" "3 2 4" "4 2 3" "4 4 3" "4 2 5" "3 4 4"; do
  set -- $v
  tag="ex_k$1_u$2_m$3"
  rm -rf build_$tag; mkdir -p build_$tag
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
    -Xcompiler -fPIC -I../../include -DTFB_EXACT_K=$1 -DTFB_EXACT_U=$2 -DTFB_EXACT_MINB=$3 -c exact.cu -o build_$tag/exact.o &
done
wait
for v in "4 2 4" "4 4 4" "4 1 4" "3 2 4" "4 2 3" "4 4 3" "4 2 5" "3 4 4"; do
  set -- $v
  tag="ex_k$1_u$2_m$3"
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../variants/libtwofold_b200_$tag.so \
    build/reduce.o build/misc.o build/host.o build_$tag/exact.o -lpthread
  rm -rf build_$tag
done
ls ../variants
