cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi0.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_r2a.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "bench rc=$?" >> gpurun_out/bench_r2a.err
