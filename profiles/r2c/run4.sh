#!/bin/bash
cd $GRAFT_REPO_ROOT
for b in 1 0; do echo "PL_BATCH_F32_BLK=$b"; PL_BATCH_F32_BLK=$b timeout 600 python profiles/r2c/c3_blk.py; done > gpurun_out/r2c_c3.txt 2>&1
cat gpurun_out/r2c_c3.txt
