#!/bin/bash
# block engine v3 (CTA-level chunk ring, tile-major layout): parity + timing + probes, each under a timeout
cd $GRAFT_REPO_ROOT
PL_BLK=1 timeout 300 python profiles/r2c/blk_check.py > gpurun_out/blk3_check.txt 2>&1
echo "exit $?" >> gpurun_out/blk3_check.txt
tail -9 gpurun_out/blk3_check.txt
for h in 1 2 3; do echo "hints $h"; PL_BLK=1 PL_BLK_HINTS=$h timeout 120 python profiles/r2c/blk_time.py c4 c5; done > gpurun_out/blk3_probe.txt 2>&1
cat gpurun_out/blk3_probe.txt
