cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2c.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_r2c.log
python profiles/r2/cold_probe.py > gpurun_out/cold_probe2.txt 2>&1
timeout 600 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_r2c.json 2> gpurun_out/bench_r2c.err
