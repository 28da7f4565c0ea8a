cd $GRAFT_REPO_ROOT
L=paper_1802_02779_b200/libpermlab_b200.so
PL_LAYER_KERNEL=lean timeout 300 python profiles/r2b/ab_lib.py $L c4 c5 >> gpurun_out/lean5.txt 2>&1
PL_LAYER_KERNEL=ws timeout 300 python profiles/r2b/ab_lib.py $L c4 c5 >> gpurun_out/lean5.txt 2>&1
PL_LAYER_KERNEL=lean timeout 300 python profiles/r2b/ab_lib.py $L c4 c5 --fma >> gpurun_out/lean5.txt 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/lean5_pytest.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c4_launches_lean.csv python profiles/r2b/ab_lib.py $L c4 --reps 1 > /dev/null 2>&1
