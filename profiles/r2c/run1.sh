#!/bin/bash
# first run of the register-blocked engine: parity + timing, old engine beside it
mkdir -p gpurun_out
timeout 900 python profiles/r2c/blk_check.py > gpurun_out/blk_check.txt 2>&1
echo "exit $?" >> gpurun_out/blk_check.txt
PL_BLK=0 timeout 600 python profiles/r2c/blk_check.py > gpurun_out/blk_check_off.txt 2>&1
tail -8 gpurun_out/blk_check.txt; tail -6 gpurun_out/blk_check_off.txt
