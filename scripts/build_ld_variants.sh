# Tuning builds of the streaming-load cache hints (TFB_LD_HINT) into paper_1401_0248_b200/variants/.
set -e
cd "$(dirname "$0")/../paper_1401_0248_b200/csrc"
mkdir -p ../variants
build() {
  tag=$1; hint=$2
  rm -rf build_$tag; mkdir -p build_$tag
  for f in reduce misc exact host; do
    nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
      -Xcompiler -fPIC -I../../include "-DTFB_LD_HINT=\"$hint\"" -c $f.cu -o build_$tag/$f.o &
  done
  wait
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o ../variants/libtwofold_b200_$tag.so build_$tag/*.o -lpthread
  rm -rf build_$tag
}
build ld_nohint ".L1::no_allocate"
build ld_128b ".L1::no_allocate.L2::128B"
build ld_evfirst ".L1::no_allocate.L2::evict_first.L2::256B"
ls ../variants
