#!/bin/bash
cd $GRAFT_REPO_ROOT
export PL_BLK=1
for g in 1 2 5; do
  echo "== debug build, grid $g"; PL_NATIVE_LIB=profiles/_variants/dbg.so PL_BLK_GRID=$g timeout 120 python profiles/r2c/blk_small.py 16 17 2>&1 | grep -v "^cta0 warp" | tail -6
done > gpurun_out/blk3_dbg.txt 2>&1
cat gpurun_out/blk3_dbg.txt
timeout 600 python profiles/r2c/blk_check.py > gpurun_out/blk3_check.txt 2>&1
echo "exit $?" >> gpurun_out/blk3_check.txt
tail -9 gpurun_out/blk3_check.txt
for h in 1 2 3; do echo "hints $h"; PL_BLK_HINTS=$h timeout 120 python profiles/r2c/blk_time.py c4 c5; done > gpurun_out/blk3_probe.txt 2>&1
cat gpurun_out/blk3_probe.txt
