cd $GRAFT_REPO_ROOT
python profiles/time_configs.py c4 c5 > gpurun_out/time8.txt 2>&1
./tests/cpp/test_permanent_device > gpurun_out/cpp8.txt 2>&1; echo "cpp rc=$?" >> gpurun_out/cpp8.txt
