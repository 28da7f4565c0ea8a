cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi18.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2b18.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_r2b18.log
timeout 300 ./tests/cpp/test_permanent_device > gpurun_out/cpp_r2b18.txt 2>&1; echo "cpp rc=$?" >> gpurun_out/cpp_r2b18.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r2b18.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r2b18.txt
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2b18.json 2> gpurun_out/bench_r2b18.err; echo "bench rc=$?" >> gpurun_out/bench_r2b18.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_r2b18.json 2>&1
