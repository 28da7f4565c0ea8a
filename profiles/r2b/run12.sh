cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -k "c3 or int_orders or pair_kernel or f32_pack or goldens or overflow" > gpurun_out/f32_12.txt 2>&1
for v in 1 0; do PL_BATCH_F32=$v python profiles/time_configs.py c3 >> gpurun_out/f32_12.txt 2>&1; done
