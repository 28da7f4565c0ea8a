#!/bin/bash
# shared-memory pipe of the ws kernel: C5 k = 16 and C4 k = 13 (full captures, raw L1TEX / shared metrics kept as text)
set -u
cd $GRAFT_REPO_ROOT
python profiles/r2b/all_configs.py c4 c5 > gpurun_out/r2c3_plain.txt 2>&1 || exit 1
ncu --set full --clock-control none -k regex:sz_ws_kernel -s 9 -c 1 -o gpurun_out/r2c3_c5 python profiles/r2b/all_configs.py c5 > gpurun_out/r2c3_ncu_c5.log 2>&1
ncu --set full --clock-control none -k regex:sz_ws_kernel -s 10 -c 1 -o gpurun_out/r2c3_c4 python profiles/r2b/all_configs.py c4 > gpurun_out/r2c3_ncu_c4.log 2>&1
for c in c5 c4; do
  ncu -i gpurun_out/r2c3_$c.ncu-rep --page raw --csv > gpurun_out/r2c3_${c}_raw.csv 2>/dev/null
  python - $c <<'PY'
import csv, sys
c = sys.argv[1]
rows = list(csv.reader(open(f"gpurun_out/r2c3_{c}_raw.csv")))
hdr, units, vals = rows[0], rows[1], rows[2]
keep = ("l1tex__data", "shared", "smem", "l1tex__throughput", "l1tex__lsu", "gpu__time_duration", "sm__cycles_elapsed.max",
        "sm__cycles_active.avg", "smsp__inst_executed.sum", "pipe_lsu", "l1tex__m_", "l1tex__f_", "Function Name", "launch__grid")
with open(f"gpurun_out/r2c3_{c}_smem.txt", "w") as f:
    for h, u, v in zip(hdr, units, vals):
        if any(k in h for k in keep):
            f.write(f"{h}\t{v}\t{u}\n")
PY
done
rm -f gpurun_out/r2c3_*.ncu-rep gpurun_out/r2c3_*_raw.csv
wc -l gpurun_out/r2c3_*_smem.txt
