cd $GRAFT_REPO_ROOT
python profiles/r2b/all_configs.py c5 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sz_ws_kernel -s 9 -c 1 \
      -o gpurun_out/r2_full_c5 python profiles/r2b/all_configs.py c5 > gpurun_out/r2_ncu_c5.log 2>&1
