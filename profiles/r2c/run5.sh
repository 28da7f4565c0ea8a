#!/bin/bash
# full validation of the tree: GPU tests, smoke, bench (own arm + reference arm)
cd $GRAFT_REPO_ROOT
timeout 3000 python -m pytest tests -m gpu -x -q > gpurun_out/r2c_gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2c_gpu_tests.log
tail -5 gpurun_out/r2c_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2c_smoke.txt 2>&1; tail -2 gpurun_out/r2c_smoke.txt
timeout 1500 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo "bench rc $?"
timeout 900 python bench.py --impl reference > gpurun_out/r2c_bench_reference.json 2> gpurun_out/r2c_bench_reference.err; echo "ref rc $?"
head -c 3000 gpurun_out/r2c_bench.json
