# rows_mis_kernel batch-depth variants (TFB_MIS_BATCH) into csrc/build/variants/, for TFB_LIB A/B runs.
set -e
cd "$(dirname "$0")/../paper_1401_0248_b200/csrc"
mkdir -p build/variants
for b in "$@"; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
    -lineinfo -Xcompiler -fPIC -I../../include -DTFB_MIS_BATCH=$b -c reduce.cu -o build/variants/reduce_mb$b.o &
done
wait
for b in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/variants/libtfb_mb$b.so \
    build/variants/reduce_mb$b.o build/misc.o build/exact.o build/host.o build/canary.o -Xlinker -z,defs -lpthread -ldl -lrt
done
ls build/variants
