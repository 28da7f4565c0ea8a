#!/bin/bash
# FP32 pack kernel: predicated adds for 0/1 packs (default build) against expanded byte coefficients (variant)
cd $GRAFT_REPO_ROOT
{
for r in 1 2; do
  echo "bit coefficients"; timeout 600 python profiles/r2c/c3_blk.py | tail -5
  echo "byte coefficients"; PL_NATIVE_LIB=profiles/_variants/nobit.so timeout 600 python profiles/r2c/c3_blk.py | tail -1
done
python - <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, paper_1802_02779_b200 as pl
from oracle import oracle as O
from paper_1802_02779_b200 import configs
for n in (10, 11, 12, 13, 14):
    a = configs.int_matrices(n, 61, seed=500 + n, lo=0, hi=2)   # 0/1
    print(n, "0/1", np.array_equal(pl.store_zechin_permanent_batch(a), O.sz_batch(a)))
    a[9, 0, 0] = 2                                                 # one pack leaves 0/1
    a[30] = 0
    print(n, "mixed", np.array_equal(pl.store_zechin_permanent_batch(a), O.sz_batch(a)))
PY
} > gpurun_out/c3_bit.txt 2>&1
cat gpurun_out/c3_bit.txt
