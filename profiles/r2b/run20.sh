cd $GRAFT_REPO_ROOT
rm -rf gpurun_out/keep gpurun_out/summ
python profiles/r2b/all_configs.py c4 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sz_ws_kernel -s 13 -c 1 \
      -o gpurun_out/r2_full_c4 python profiles/r2b/all_configs.py c4 > gpurun_out/r2_ncu_c4.log 2>&1
