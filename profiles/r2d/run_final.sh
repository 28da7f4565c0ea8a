#!/bin/bash
# final validation of the tree: GPU tests, smoke, bench (reference arm + own arm), ncu launch list of one call per config
cd $GRAFT_REPO_ROOT
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2d_gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2d_gpu_tests.log
tail -4 gpurun_out/r2d_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2d_smoke.txt 2>&1; tail -1 gpurun_out/r2d_smoke.txt
timeout 900 python bench.py --impl reference > gpurun_out/r2d_bench_reference.json 2> gpurun_out/r2d_bench_reference.err; echo "ref rc $?"
timeout 1500 python bench.py > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "bench rc $?"
python profiles/r2b/all_configs.py > gpurun_out/r2d_plain.txt 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --cache-control none --csv --log-file gpurun_out/r2d_launches.csv python profiles/r2b/all_configs.py > /dev/null 2>&1
mkdir -p gpurun_out/summ_r2d && SUMMARY_DIR=gpurun_out/summ_r2d python profiles/summarize.py r2d gpurun_out/r2d_launches.csv > gpurun_out/summ_r2d/log.txt 2>&1
ls gpurun_out/summ_r2d
