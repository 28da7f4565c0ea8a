cd $GRAFT_REPO_ROOT
L=paper_1802_02779_b200/libpermlab_b200.so
for K in ws lean; do
  echo "== $K default" >> gpurun_out/graph7.txt; PL_LAYER_KERNEL=$K python profiles/r2b/ab_lib.py $L c4 >> gpurun_out/graph7.txt 2>&1
  echo "== $K graph" >> gpurun_out/graph7.txt; PL_LAYER_KERNEL=$K python profiles/r2b/ab_lib.py $L c4 --graph >> gpurun_out/graph7.txt 2>&1
  echo "== $K nopdl" >> gpurun_out/graph7.txt; PL_WS_PDL=0 PL_LAYER_KERNEL=$K python profiles/r2b/ab_lib.py $L c4 >> gpurun_out/graph7.txt 2>&1
done
