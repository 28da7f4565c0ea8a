#!/bin/bash
# FP32 pack kernel with byte coefficients + two-term table words
cd $GRAFT_REPO_ROOT
{
for r in 1 2; do timeout 600 python profiles/r2c/c3_blk.py | tail -4; done
python - <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, paper_1802_02779_b200 as pl
from oracle import oracle as O
from paper_1802_02779_b200 import configs
for n in (10, 11, 12, 13, 14):
    a = configs.int_matrices(n, 61, seed=500 + n, lo=0, hi=2)
    a[7, 0, 0] = 200; a[8, 1, 1] = -129; a[20, 2, 2] = 127; a[21, 3, 3] = -128
    print(n, np.array_equal(pl.store_zechin_permanent_batch(a), O.sz_batch(a)))
    b = configs.int_matrices(n, 64, seed=900 + n, lo=-1, hi=2)
    print(n, np.array_equal(pl.store_zechin_permanent_batch(b), O.sz_batch(b)))
PY
} > gpurun_out/c3_byte2.txt 2>&1
cat gpurun_out/c3_byte2.txt
