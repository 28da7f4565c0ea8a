#!/bin/bash
# block engine v2 variants: ring slots x CTAs per SM (tables for the header binomials in all)
cd $GRAFT_REPO_ROOT
export PL_BLK=1
{
echo "default (3 slots, 4 CTAs)"; python profiles/r2c/blk_time.py c4 c5
for v in s2 s4 s4c3 s6c3; do
  for c in 3 4; do
    echo "variant $v PL_BLK_CTAS=$c"; PL_BLK_CTAS=$c PL_NATIVE_LIB=profiles/_variants/$v.so python profiles/r2c/blk_time.py c4 c5
  done
done
} > gpurun_out/blk_variants.txt 2>&1
cat gpurun_out/blk_variants.txt
