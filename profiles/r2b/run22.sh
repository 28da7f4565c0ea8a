cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "c3 or int_orders or pair_kernel or f32_pack" > gpurun_out/cols22.txt 2>&1
for v in "" rows q2 q8; do
  echo "== $v" >> gpurun_out/cols22.txt
  if [ -n "$v" ]; then PL_NATIVE_LIB=profiles/_variants/$v.so python profiles/time_configs.py c3 >> gpurun_out/cols22.txt 2>&1; else python profiles/time_configs.py c3 >> gpurun_out/cols22.txt 2>&1; fi
done
