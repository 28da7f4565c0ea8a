#!/bin/bash
# Round-2 profile captures (GPU box, via gpurun). Every command runs once
# without ncu first; ncu only after it exits 0. Launch list: unlocked clocks
# and no cache flush between kernels (--clock-control none --cache-control
# none), so per-launch times compare with the bench's steps.
set -u
cd $GRAFT_REPO_ROOT
T=r2
python profiles/r2b/all_configs.py > gpurun_out/${T}_plain.txt 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --cache-control none --csv --log-file gpurun_out/${T}_launches.csv python profiles/r2b/all_configs.py > /dev/null 2>&1
full() {  # full capture: name, kernel regex, skip count, config
  ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
      -o gpurun_out/${T}_full_$1 python profiles/r2b/all_configs.py $4 > gpurun_out/${T}_ncu_$1.log 2>&1
}
full c2 sz_batch_tma 1 c2
full c3 sz_batch_f32_pack 1 c3
full c4 sz_ws_kernel 13 c4          # second call (9 ws layers k=9..17 per call): k=13
full c4lean sz_lean_kernel 16 c4    # second call's k=5 (first call: 15 lean layers)
full c5 sz_ws_kernel 9 c5           # ws layers k=7..25: k=16 of the first call
python - > gpurun_out/${T}_b16.txt 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_1802_02779_b200 as pl
a = torch.from_numpy(np.random.default_rng(16).standard_normal((2000, 16, 16)) + 0j).cuda()
pl.store_zechin_permanent_batch(a); torch.cuda.synchronize(); print("ok")
PY
ncu --set full --clock-control none --import-source on -k regex:sz_lean_kernel -s 5 -c 1 -o gpurun_out/${T}_full_b16 \
    python - > gpurun_out/${T}_ncu_b16.log 2>&1 <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, torch, paper_1802_02779_b200 as pl
a = torch.from_numpy(np.random.default_rng(16).standard_normal((2000, 16, 16)) + 0j).cuda()
pl.store_zechin_permanent_batch(a); torch.cuda.synchronize(); print("ok")
PY
ls -la gpurun_out/ | grep ${T}_
# summaries on the box (the .ncu-rep files are too large to travel back together)
mkdir -p gpurun_out/summ
SUMMARY_DIR=gpurun_out/summ python profiles/summarize.py r2 gpurun_out/r2_launches.csv gpurun_out/r2_full_*.ncu-rep
for f in gpurun_out/r2_full_*.ncu-rep; do
  b=$(basename $f .ncu-rep)
  k=$(ncu -i $f --page raw --csv 2>/dev/null | python -c "import csv,sys; r=list(csv.reader(sys.stdin)); print(dict(zip(r[0],r[2])).get('Function Name','')[:40])")
  python profiles/linestats.py $f "${k%%<*}" > gpurun_out/summ/${b}_lines.txt 2>&1
done
mkdir -p gpurun_out/keep && mv gpurun_out/r2_full_c5.ncu-rep gpurun_out/keep/ 2>/dev/null
rm -f gpurun_out/r2_full_*.ncu-rep
