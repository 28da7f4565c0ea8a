cd $GRAFT_REPO_ROOT
for L in paper_1802_02779_b200/libpermlab_b200.so profiles/_variants/old_d3e.so; do
  echo "== $L default" >> gpurun_out/pdl4.txt; python profiles/r2b/ab_lib.py $L c4 >> gpurun_out/pdl4.txt 2>&1
  echo "== $L nopdl" >> gpurun_out/pdl4.txt; PL_WS_PDL=0 python profiles/r2b/ab_lib.py $L c4 >> gpurun_out/pdl4.txt 2>&1
  echo "== $L graph" >> gpurun_out/pdl4.txt; python profiles/r2b/ab_lib.py $L c4 --graph >> gpurun_out/pdl4.txt 2>&1
done
