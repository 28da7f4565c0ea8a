cd $GRAFT_REPO_ROOT
PL_COLD_LOG=1 python profiles/r2b/cold_c4.py > gpurun_out/cold19.txt 2>&1
CUDA_MODULE_LOADING=EAGER PL_COLD_LOG=1 python profiles/r2b/cold_c4.py >> gpurun_out/cold19.txt 2>&1
python bench.py --cold-call c4 >> gpurun_out/cold19.txt 2>&1
