cd $GRAFT_REPO_ROOT
python profiles/time_configs.py c4 c5 > gpurun_out/time7.txt 2>&1
python profiles/r2/cold_probe.py >> gpurun_out/time7.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "parity or shard or c4 or c5" > gpurun_out/gputest_r2d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_r2d.log
