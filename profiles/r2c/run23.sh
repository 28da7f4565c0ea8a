#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2c_gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2c_gpu_tests.log
tail -4 gpurun_out/r2c_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
