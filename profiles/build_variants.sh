#!/bin/bash
# Build tuning variants of the device library for A/B timing:
#   profiles/build_variants.sh name "-DPL_WS_D16=13 -DPL_WS_NSG16=3" [...]
# capi.cu (layer kernels) and batch.cu (batch kernels) are compiled with the
# flags; the other objects come from the default build.
# Output: profiles/_variants/<name>.so (git-ignored); select with PL_NATIVE_LIB=<path>.
set -e
cd "$(dirname "$0")/.."
mkdir -p profiles/_variants
make build/boson.o build/multi.o build/ryser.o build/blk.o > /dev/null
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
while [ $# -ge 2 ]; do
  ( $NV $2 -c -o profiles/_variants/$1.capi.o paper_1802_02779_b200/csrc/capi.cu &&
    $NV $2 -c -o profiles/_variants/$1.batch.o paper_1802_02779_b200/csrc/batch.cu &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o profiles/_variants/$1.so profiles/_variants/$1.capi.o \
         profiles/_variants/$1.batch.o build/boson.o build/multi.o build/ryser.o build/blk.o -lcudart -ldl &&
    rm -f profiles/_variants/$1.capi.o profiles/_variants/$1.batch.o ) &
  shift 2
done
wait
