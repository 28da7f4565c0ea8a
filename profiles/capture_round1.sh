#!/bin/bash
# Round-1 profile captures (run on the GPU box via gpurun). Each command runs
# once without ncu first; ncu only after it exits 0.
set -u
mkdir -p gpurun_out
./profiles/microbench > gpurun_out/microbench.json 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/r1_plain.json 2> gpurun_out/r1_plain.err && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/r1_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
for c in c2 c3 c4; do
  python profiles/run_config.py $c > /dev/null 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:sz_ -s 12 -c 1 \
        -o gpurun_out/r1_full_$c python profiles/run_config.py $c > /dev/null 2>&1
done
python profiles/run_config.py c5 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sz_ws -s 13 -c 1 \
      -o gpurun_out/r1_full_c5 python profiles/run_config.py c5 > /dev/null 2>&1
ls -la gpurun_out/
