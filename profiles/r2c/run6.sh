#!/bin/bash
# block engine v2 (TMA stream rings): parity + timing + probes
cd $GRAFT_REPO_ROOT
PL_BLK=1 timeout 900 python profiles/r2c/blk_check.py > gpurun_out/blk2_check.txt 2>&1
echo "exit $?" >> gpurun_out/blk2_check.txt
tail -9 gpurun_out/blk2_check.txt
for h in 1 2 3; do echo "hints $h"; PL_BLK=1 PL_BLK_HINTS=$h timeout 300 python profiles/r2c/blk_time.py c4 c5; done > gpurun_out/blk2_probe.txt 2>&1
cat gpurun_out/blk2_probe.txt
