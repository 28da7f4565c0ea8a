#!/bin/bash
# ws kernel, complex low-term coefficients: split re/im arrays (default build) against 16-byte gathers (variant)
cd $GRAFT_REPO_ROOT
{
for r in 1 2 3; do
  echo "split"; python profiles/r2c/blk_time.py c5
  echo "nosplit"; PL_NATIVE_LIB=profiles/_variants/nosplit.so python profiles/r2c/blk_time.py c5
done
echo "batch n=16 c128 (lean kernel unaffected) / n=20 c128 single"
python - <<'PY'
import sys; sys.path.insert(0, '.')
import numpy as np, paper_1802_02779_b200 as pl
from oracle import oracle as O
from paper_1802_02779_b200 import configs
for n in (19, 21, 23):
    c = configs.complex_uniform((n, n), seed=2000 + n)
    v = complex(pl.store_zechin_permanent(c).value); w = complex(O.sz_batch(c[None])[0])
    print(n, v == w, v)
PY
} > gpurun_out/coef_split.txt 2>&1
cat gpurun_out/coef_split.txt
