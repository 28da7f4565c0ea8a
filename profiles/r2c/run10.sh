#!/bin/bash
# full GPU test suite of the tree
cd $GRAFT_REPO_ROOT
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2c_gpu_tests.log 2>&1; echo "pytest rc $?" >> gpurun_out/r2c_gpu_tests.log
tail -6 gpurun_out/r2c_gpu_tests.log
