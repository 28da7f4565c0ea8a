cd $GRAFT_REPO_ROOT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  for w in f32 lean ws ryser overlap; do
    echo "== $tool $w" >> gpurun_out/san30.txt
    timeout 600 $CS --tool $tool --error-exitcode 9 python profiles/r2b/sanitize_cases.py $w 2>&1 | grep -E "ERROR SUMMARY|error|Error|ok|pack|lean|ws|ryser" | tail -4 >> gpurun_out/san30.txt
  done
done
