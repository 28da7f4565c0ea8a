cd $GRAFT_REPO_ROOT
nproc > gpurun_out/nproc.txt; free -g >> gpurun_out/nproc.txt
timeout 900 python bench.py --cpu-large-only > gpurun_out/cpu_large.json 2> gpurun_out/cpu_large.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r2b.json 2> gpurun_out/bench_r2b.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_r2b_ref.json 2>&1
