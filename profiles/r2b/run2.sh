cd $GRAFT_REPO_ROOT
for i in 1 2; do
python profiles/r2b/ab_lib.py paper_1802_02779_b200/libpermlab_b200.so c4 c5 >> gpurun_out/ab2.txt 2>&1
python profiles/r2b/ab_lib.py profiles/_variants/old_d3e.so c4 c5 >> gpurun_out/ab2.txt 2>&1
done
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c4_launches_new.csv python profiles/r2b/ab_lib.py paper_1802_02779_b200/libpermlab_b200.so c4 --reps 1 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/c4_launches_old.csv python profiles/r2b/ab_lib.py profiles/_variants/old_d3e.so c4 --reps 1 > /dev/null 2>&1
