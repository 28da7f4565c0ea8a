#!/bin/bash
# Per-layer kernel time and DRAM bytes of one C5 (or C4) evaluation:
#   profiles/layer_times.sh c5 out.csv  [extra env via the caller]
cfg=${1:-c5}; out=${2:-gpurun_out/layers_$cfg.csv}
mkdir -p "$(dirname "$out")"
# time_configs runs 2 warm-ups + reps; skip the warm-up evaluations' launches
n=$([ "$cfg" = c5 ] && echo 29 || echo 23)
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:sz_ws_kernel --launch-skip $((2 * n)) --launch-count $n --csv --log-file "$out" \
    python profiles/time_configs.py $cfg > /dev/null 2>&1
