cd $GRAFT_REPO_ROOT
for v in "" per4 per4b2 per1; do
  L=paper_1802_02779_b200/libpermlab_b200.so; [ -n "$v" ] && L=profiles/_variants/$v.so
  echo "== $v all-lean" >> gpurun_out/per26.txt
  PL_LAYER_KERNEL=lean python profiles/r2b/ab_lib.py $L c4 >> gpurun_out/per26.txt 2>&1
  echo "== $v hybrid" >> gpurun_out/per26.txt
  python profiles/r2b/ab_lib.py $L c4 >> gpurun_out/per26.txt 2>&1
done
