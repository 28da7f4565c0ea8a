cd $GRAFT_REPO_ROOT
for h in 0x905 0x105905 0x205905 0x405905 0x805905 0x1005905 0x2005905; do
  echo "hints $h" >> gpurun_out/qcap3.txt
  PL_WS_HINTS=$h python profiles/r2b/ab_lib.py paper_1802_02779_b200/libpermlab_b200.so c4 c5 >> gpurun_out/qcap3.txt 2>&1
done
