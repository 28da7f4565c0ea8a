cd $GRAFT_REPO_ROOT
./profiles/r2/alloc_probe > gpurun_out/alloc_probe.txt 2>&1
python profiles/r2/cold_probe.py > gpurun_out/cold_probe.txt 2>&1
python profiles/r2/cold_probe.py >> gpurun_out/cold_probe.txt 2>&1
