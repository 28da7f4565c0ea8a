cd $GRAFT_REPO_ROOT
python profiles/r2b/all_configs.py > gpurun_out/r2_plain.txt 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --cache-control none --csv --log-file gpurun_out/r2_launches.csv python profiles/r2b/all_configs.py > /dev/null 2>&1
mkdir -p gpurun_out/summ && SUMMARY_DIR=gpurun_out/summ python profiles/summarize.py r2 gpurun_out/r2_launches.csv
