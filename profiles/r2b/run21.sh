cd $GRAFT_REPO_ROOT
for i in 1 2; do
for v in "" ps256 ps1k pub1k both; do
  echo "== $v" >> gpurun_out/sleep21.txt
  L=paper_1802_02779_b200/libpermlab_b200.so; [ -n "$v" ] && L=profiles/_variants/$v.so
  python profiles/r2b/ab_lib.py $L c4 c5 >> gpurun_out/sleep21.txt 2>&1
done; done
