cd $GRAFT_REPO_ROOT
L=paper_1802_02779_b200/libpermlab_b200.so
ncu --set full --clock-control none --import-source on -k regex:sz_lean -s 10 -c 1 -o gpurun_out/lean_c4_k13 \
   python profiles/r2b/ab_lib.py $L c4 --reps 1 > gpurun_out/ncu6.log 2>&1
