cd $GRAFT_REPO_ROOT
L=paper_1802_02779_b200/libpermlab_b200.so
PL_LAYER_KERNEL=ws python profiles/r2b/ab_lib.py $L c4 >> gpurun_out/host8.txt 2>&1
python profiles/r2b/ab_lib.py profiles/_variants/old_d3e.so c4 >> gpurun_out/host8.txt 2>&1
