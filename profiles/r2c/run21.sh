#!/bin/bash
# FP32 pack kernel, 0/1 packs: 16-bit layers k <= 8 (default build, 5 CTAs per SM) against variants
cd $GRAFT_REPO_ROOT
{
for r in 1 2; do
  echo "u16 layers, min 5 CTAs (default)"; timeout 600 python profiles/r2c/c3_blk.py | tail -5
  for v in nou16 u16r64 u16c6; do echo "variant $v"; PL_NATIVE_LIB=profiles/_variants/$v.so timeout 600 python profiles/r2c/c3_blk.py | tail -1; done
done
python - <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, paper_1802_02779_b200 as pl
from oracle import oracle as O
from paper_1802_02779_b200 import configs
for n in (10, 11, 12, 13, 14):
    a = configs.int_matrices(n, 61, seed=500 + n, lo=0, hi=2)   # 0/1
    a[3] = np.triu(np.ones((n, n), dtype=np.int64))             # dense upper triangle: per = 1, big intermediates
    print(n, "0/1", np.array_equal(pl.store_zechin_permanent_batch(a), O.sz_batch(a)))
    b = np.ones((8, n, n), dtype=np.int64); b[:, np.arange(n), np.arange(n)] = 0   # derangement counts: the largest 0/1 values that still pass the FP32 bound or fall back
    print(n, "ones-minus-identity", np.array_equal(pl.store_zechin_permanent_batch(b), O.sz_batch(b)))
PY
} > gpurun_out/c3_u16.txt 2>&1
cat gpurun_out/c3_u16.txt
