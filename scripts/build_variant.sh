# A tuning variant of the library with extra -D flags (reduce.cu only; the other objects
# from csrc/build/), into csrc/build/variants/libtfb_<name>.so for TFB_LIB A/B runs:
#   bash scripts/build_variant.sh NAME "-DTFB_X=1 -DTFB_Y=2" [NAME2 "FLAGS2" ...]
set -e
cd "$(dirname "$0")/../paper_1401_0248_b200/csrc"
make -s
mkdir -p build/variants
args=("$@")
for ((i = 0; i < ${#args[@]}; i += 2)); do
  name=${args[i]}; flags=${args[i+1]}
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -ftz=false -prec-div=true -prec-sqrt=true \
    -lineinfo -Xcompiler -fPIC -I../../include $flags -c reduce.cu -o build/variants/reduce_$name.o &
done
wait
for ((i = 0; i < ${#args[@]}; i += 2)); do
  name=${args[i]}
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o build/variants/libtfb_$name.so \
    build/variants/reduce_$name.o $(ls build/*.o | grep -v '/reduce.o$') -Xlinker -z,defs -lpthread -ldl -lrt
  rm -f build/variants/reduce_$name.o
done
ls build/variants
