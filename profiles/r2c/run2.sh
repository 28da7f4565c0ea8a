#!/bin/bash
# ncu of the register-blocked engine on C4: launch list and a full capture of super-layer j = 10
set -u
cd $GRAFT_REPO_ROOT
T=r2c
python profiles/r2b/all_configs.py c4 > gpurun_out/${T}_plain.txt 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --cache-control none --csv --log-file gpurun_out/${T}_launches.csv python profiles/r2b/all_configs.py c4 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sz_blk_kernel -s 32 -c 1 \
    -o gpurun_out/${T}_full_c4 python profiles/r2b/all_configs.py c4 > gpurun_out/${T}_ncu_c4.log 2>&1
mkdir -p gpurun_out/summ
SUMMARY_DIR=gpurun_out/summ python profiles/summarize.py ${T} gpurun_out/${T}_launches.csv gpurun_out/${T}_full_c4.ncu-rep > gpurun_out/summ/log.txt 2>&1
python profiles/linestats.py gpurun_out/${T}_full_c4.ncu-rep sz_blk_kernel > gpurun_out/summ/${T}_full_c4_lines.txt 2>&1
ls -la gpurun_out gpurun_out/summ
