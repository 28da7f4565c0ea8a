cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q > gpurun_out/b17.txt 2>&1
python - >> gpurun_out/b17.txt 2>&1 <<'PY'
import sys, time, os; sys.path.insert(0, '.')
import numpy as np, torch, paper_1802_02779_b200 as pl
for n, cnt in ((16, 2000), (18, 500), (20, 200)):
    a = torch.from_numpy(np.random.default_rng(n).standard_normal((cnt, n, n)) + 0j).cuda()
    pl.store_zechin_permanent_batch(a); torch.cuda.synchronize()
    t = time.perf_counter(); pl.store_zechin_permanent_batch(a); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"n={n} x{cnt} c128 batch: {dt*1e3:.2f} ms, {cnt/dt:.0f} perm/s")
PY
PL_BATCH_LAYERS=0 python - >> gpurun_out/b17.txt 2>&1 <<'PY'
import sys, time, os; sys.path.insert(0, '.')
import numpy as np, torch, paper_1802_02779_b200 as pl
for n, cnt in ((16, 2000), (18, 500), (20, 200)):
    a = torch.from_numpy(np.random.default_rng(n).standard_normal((cnt, n, n)) + 0j).cuda()
    pl.store_zechin_permanent_batch(a); torch.cuda.synchronize()
    t = time.perf_counter(); pl.store_zechin_permanent_batch(a); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"PER-MATRIX n={n} x{cnt} c128 batch: {dt*1e3:.2f} ms, {cnt/dt:.0f} perm/s")
PY
