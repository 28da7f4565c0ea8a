#!/bin/bash
# ncu full capture of block engine v2, super-layer j = 10 of C4
set -u
cd $GRAFT_REPO_ROOT
export PL_BLK=1
T=r2c2
python profiles/r2b/all_configs.py c4 > gpurun_out/${T}_plain.txt 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:sz_blk_kernel -s 32 -c 1 \
    -o gpurun_out/${T}_full_c4 python profiles/r2b/all_configs.py c4 > gpurun_out/${T}_ncu_c4.log 2>&1
mkdir -p gpurun_out/summ
SUMMARY_DIR=gpurun_out/summ python profiles/summarize.py ${T} gpurun_out/${T}_full_c4.ncu-rep > gpurun_out/summ/log.txt 2>&1
python profiles/linestats.py gpurun_out/${T}_full_c4.ncu-rep sz_blk_kernel > gpurun_out/summ/${T}_full_c4_lines.txt 2>&1
rm -f gpurun_out/${T}_full_c4.ncu-rep
