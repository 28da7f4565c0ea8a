#!/bin/bash
# Round-1 profile captures (run on the GPU box via gpurun). Each command runs
# once without ncu first; ncu only after it exits 0.
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
./profiles/microbench > gpurun_out/microbench.json 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1
# batched kernels: the single sz_batch launch of one API call; c4: a middle layer (k=14)
python profiles/run_config.py c2 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sz_batch -c 1 \
      -o gpurun_out/${TAG}_full_c2 python profiles/run_config.py c2 > /dev/null 2>&1
python profiles/run_config.py c3 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sz_batch -c 1 \
      -o gpurun_out/${TAG}_full_c3 python profiles/run_config.py c3 > /dev/null 2>&1
python profiles/run_config.py c4 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sz_ws -s 10 -c 1 \
      -o gpurun_out/${TAG}_full_c4 python profiles/run_config.py c4 > /dev/null 2>&1
python profiles/run_config.py c5 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sz_ws -s 13 -c 1 \
      -o gpurun_out/${TAG}_full_c5 python profiles/run_config.py c5 > /dev/null 2>&1
ls -la gpurun_out/ | grep ${TAG}
