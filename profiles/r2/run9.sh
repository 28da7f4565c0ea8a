cd $GRAFT_REPO_ROOT
for h in 0x905 0x305905 0x605905 0xC05905 0x1805905; do
  echo "hints $h" >> gpurun_out/time9.txt
  PL_WS_HINTS=$h python profiles/time_configs.py c4 c5 >> gpurun_out/time9.txt 2>&1
done
