# Debug build of the library with device-side range/capacity assertions (TFB_DEBUG=1):
# paper_1401_0248_b200/csrc/build/debug/libtwofold_b200_debug.so, used via TFB_LIB=<path>
# (compute-sanitizer is closed on the GPU pool; this is the substitute).
# ptxas runs at -O1 here: with the assertions compiled in, ptxas -O3 (CUDA 12.9)
# mis-compiles the "LDG deep" leaves kernel (UF=2) — every leaf pair comes out
# zero and larger leaves fault — while the same source is correct at -O1 and in
# the release build (-O3, no assertions; tests/test_gpu_fuzz.py covers it).
set -e
cd "$(dirname "$0")/../paper_1401_0248_b200/csrc"
make -s   # the release objects (the host leaf reducer is reused as is)
mkdir -p build/debug
for f in reduce misc exact host canary; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -ftz=false -prec-div=true \
    -prec-sqrt=true -lineinfo -Xcompiler -fPIC -I../../include -DTFB_DEBUG=1 -Xptxas -O1 -c $f.cu -o build/debug/$f.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/debug/libtwofold_b200_debug.so \
  build/debug/reduce.o build/debug/misc.o build/debug/exact.o build/debug/host.o build/debug/canary.o \
  build/hostleaf_avx512.o build/hostleaf_base.o -Xlinker -z,defs -lpthread -ldl -lrt
rm -f build/debug/*.o
echo built build/debug/libtwofold_b200_debug.so
