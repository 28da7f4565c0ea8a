cd $GRAFT_REPO_ROOT
python profiles/time_configs.py c4 c5 > gpurun_out/time6.txt 2>&1
PL_WS_GRID=148 python profiles/time_configs.py c4 >> gpurun_out/time6.txt 2>&1
