#!/bin/bash
# Variants of the block engine (blk.cu only; the other objects from the default build):
#   profiles/r2c/build_blk_variants.sh name "-DPL_BLK_SLOTS=4" [...]  ->  profiles/_variants/<name>.so
set -e
cd "$(dirname "$0")/../.."
mkdir -p profiles/_variants
make build/capi.o build/batch.o build/boson.o build/multi.o build/ryser.o > /dev/null
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
while [ $# -ge 2 ]; do
  ( $NV $2 -c -o profiles/_variants/$1.blk.o paper_1802_02779_b200/csrc/blk.cu &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o profiles/_variants/$1.so build/capi.o build/batch.o \
         build/boson.o build/multi.o build/ryser.o profiles/_variants/$1.blk.o -lcudart -ldl &&
    rm -f profiles/_variants/$1.blk.o ) &
  shift 2
done
wait
