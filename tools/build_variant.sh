#!/bin/bash
# Build libpilc_sm100a.so with extra nvcc defines into tools/exp/<name>.so for
# A/B timing on the GPU box (PILC_LIB_PATH=tools/exp/<name>.so python ...).
#   tools/build_variant.sh <name> -DFOO=1 ...
set -e
name=$1; shift
cd "$(dirname "$0")/../paper_2206_05279_b200/csrc"
out=../../tools/exp/$name
mkdir -p "$out"
for f in api rans twar container vq tc_conv; do
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -c $f.cu -o "$out/$f.o" &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "../../tools/exp/$name.so" "$out"/*.o -lcudart
rm -rf "$out"
echo "tools/exp/$name.so"
