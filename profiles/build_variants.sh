#!/bin/bash
# Build layer-kernel geometry variants of the device library for A/B timing:
#   profiles/build_variants.sh name "-DPL_WS_D16=13 -DPL_WS_NSG16=3" [...]
# Output: profiles/_variants/<name>.so (git-ignored); select with PL_NATIVE_LIB=<path>.
set -e
cd "$(dirname "$0")/.."
mkdir -p profiles/_variants
while [ $# -ge 2 ]; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
       -Xptxas -warn-spills $2 -shared -o profiles/_variants/$1.so paper_1802_02779_b200/csrc/capi.cu -lcudart &
  shift 2
done
wait
