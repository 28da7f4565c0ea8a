cd $GRAFT_REPO_ROOT
./profiles/r2/smem_path > gpurun_out/smem_path.txt 2>&1
python profiles/run_config.py c5 > gpurun_out/c5_plain.txt 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sz_ws -s 13 -c 1 \
      -o gpurun_out/r2a_full_c5 python profiles/run_config.py c5 > gpurun_out/ncu_c5.log 2>&1
