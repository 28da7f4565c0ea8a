cd $GRAFT_REPO_ROOT
for v in 4 8; do echo "P=$v" >> gpurun_out/f32_13.txt; PL_BATCH_F32_P=$v python profiles/time_configs.py c3 >> gpurun_out/f32_13.txt 2>&1; done
PL_BATCH_F32_P=8 timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "c3 or int_orders or pair_kernel or f32_pack" >> gpurun_out/f32_13.txt 2>&1
python profiles/time_configs.py c3 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:f32_pack -s 3 -c 1 -o gpurun_out/f32_c3 python profiles/time_configs.py c3 > gpurun_out/ncu13.log 2>&1
