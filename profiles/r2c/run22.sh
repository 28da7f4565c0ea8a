#!/bin/bash
# FP32 pack kernel with byte coefficients: threads per CTA
cd $GRAFT_REPO_ROOT
{
for r in 1 2; do
  echo "256 threads (default)"; timeout 600 python profiles/r2c/c3_blk.py | tail -1
  for v in t128 t192 t384; do echo "variant $v"; PL_NATIVE_LIB=profiles/_variants/$v.so timeout 600 python profiles/r2c/c3_blk.py | tail -1; done
done
} > gpurun_out/c3_threads.txt 2>&1
cat gpurun_out/c3_threads.txt
