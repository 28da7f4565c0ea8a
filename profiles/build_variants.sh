#!/bin/bash
# Build layer-kernel geometry variants of the device library for A/B timing:
#   profiles/build_variants.sh name "-DPL_WS_D16=13 -DPL_WS_NSG16=3" [...]
# Output: profiles/_variants/<name>.so (git-ignored); select with PL_NATIVE_LIB=<path>.
set -e
cd "$(dirname "$0")/.."
mkdir -p profiles/_variants
make build/boson.o > /dev/null
while [ $# -ge 2 ]; do
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
         -Xptxas -warn-spills $2 -c -o profiles/_variants/$1.o paper_1802_02779_b200/csrc/capi.cu &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o profiles/_variants/$1.so profiles/_variants/$1.o build/boson.o -lcudart ) &
  shift 2
done
wait
