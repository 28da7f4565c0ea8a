#!/bin/bash
# timing probes of the block engine: without high terms (1), without window terms (2), neither (3)
cd $GRAFT_REPO_ROOT
for h in 0 1 2 3; do echo "hints $h"; PL_BLK_HINTS=$h python profiles/r2c/blk_time.py c4 c5; done > gpurun_out/r2c_probe.txt 2>&1
cat gpurun_out/r2c_probe.txt
