cd $GRAFT_REPO_ROOT
L=paper_1802_02779_b200/libpermlab_b200.so
for K in hybrid ws lean; do
  if [ $K = hybrid ]; then unset PL_LAYER_KERNEL; else export PL_LAYER_KERNEL=$K; fi
  echo "== $K default" >> gpurun_out/hyb9.txt; python profiles/r2b/ab_lib.py $L c4 c5 >> gpurun_out/hyb9.txt 2>&1
  echo "== $K graph" >> gpurun_out/hyb9.txt; python profiles/r2b/ab_lib.py $L c4 --graph >> gpurun_out/hyb9.txt 2>&1
done
unset PL_LAYER_KERNEL
for mb in 8 48 96; do echo "== maxmb $mb" >> gpurun_out/hyb9.txt; PL_LEAN_MAX_MB=$mb python profiles/r2b/ab_lib.py $L c4 >> gpurun_out/hyb9.txt 2>&1; done
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/hyb9_pytest.txt 2>&1
