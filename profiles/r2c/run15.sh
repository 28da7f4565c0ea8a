#!/bin/bash
# final validation of the tree: GPU tests, smoke, bench (own arm + reference arm), ncu launch list of the bench
cd $GRAFT_REPO_ROOT
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2c_gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2c_gpu_tests.log
tail -4 gpurun_out/r2c_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2c_smoke.txt 2>&1; tail -1 gpurun_out/r2c_smoke.txt
timeout 900 python bench.py --impl reference > gpurun_out/r2c_bench_reference.json 2> gpurun_out/r2c_bench_reference.err; echo "ref rc $?"
timeout 1500 python bench.py > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo "bench rc $?"
PL_BLK=1 timeout 300 python profiles/r2c/blk_time.py c4 c5 > gpurun_out/r2c_blk_final.txt 2>&1; cat gpurun_out/r2c_blk_final.txt
