#!/bin/bash
# variant libraries: name "flags" ...
set -e
cd /root/repo
mkdir -p profiles/_variants
make build/boson.o build/multi.o build/ryser.o build/batch.o > /dev/null
while [ $# -ge 2 ]; do
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $2 -c -o profiles/_variants/$1.o paper_1802_02779_b200/csrc/capi.cu &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o profiles/_variants/$1.so profiles/_variants/$1.o build/batch.o build/boson.o build/multi.o build/ryser.o -lcudart -ldl ) &
  shift 2
done
wait
