cd $GRAFT_REPO_ROOT
for v in "" d13n6 d13n5s3 fs1n8; do
  L=paper_1802_02779_b200/libpermlab_b200.so; [ -n "$v" ] && L=profiles/_variants/$v.so
  echo "== $v" >> gpurun_out/geo27.txt
  timeout 300 python profiles/r2b/ab_lib.py $L c5 >> gpurun_out/geo27.txt 2>&1
done
