cd $GRAFT_REPO_ROOT
for v in "" profiles/_variants/t128.so profiles/_variants/t512.so; do
  echo "lib=$v" >> gpurun_out/t14.txt
  if [ -n "$v" ]; then PL_NATIVE_LIB=$v python profiles/time_configs.py c3 >> gpurun_out/t14.txt 2>&1; else python profiles/time_configs.py c3 >> gpurun_out/t14.txt 2>&1; fi
done
