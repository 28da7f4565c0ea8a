#!/bin/bash
# ncu full capture of the FP32 pack kernel with byte coefficients (C3)
set -u
cd $GRAFT_REPO_ROOT
T=r2c_c3
python profiles/r2b/all_configs.py c3 > gpurun_out/${T}_plain.txt 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:sz_batch_f32_pack -s 1 -c 1 \
    -o gpurun_out/${T}_full python profiles/r2b/all_configs.py c3 > gpurun_out/${T}_ncu.log 2>&1
mkdir -p gpurun_out/summ
SUMMARY_DIR=gpurun_out/summ python profiles/summarize.py ${T} gpurun_out/${T}_full.ncu-rep > gpurun_out/summ/log.txt 2>&1
python profiles/linestats.py gpurun_out/${T}_full.ncu-rep sz_batch_f32_pack > gpurun_out/summ/${T}_lines.txt 2>&1
ncu -i gpurun_out/${T}_full.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h,u,v=r[0],r[1],r[2]
for a,b,c in zip(h,u,v):
    if any(k in a for k in ('l1tex__data_pipe_lsu_wavefronts','l1tex__lsu_writeback_active.avg.pct','l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum','gpu__time_duration.sum')): print(a,c,b,sep='\t')
" > gpurun_out/summ/${T}_pipe.txt
rm -f gpurun_out/${T}_full.ncu-rep
