cd $GRAFT_REPO_ROOT
L=paper_1802_02779_b200/libpermlab_b200.so
python profiles/r2b/ab_lib.py $L c4 --graph >> gpurun_out/g10.txt 2>&1
python profiles/r2b/ab_lib.py $L c4 c5 --fma >> gpurun_out/g10.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/g10_pytest.txt 2>&1
./tests/cpp/test_permanent_device > gpurun_out/g10_cpp.txt 2>&1; echo "cpp rc=$?" >> gpurun_out/g10_cpp.txt
