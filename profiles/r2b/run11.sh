cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_ryser_gpu.py tests/test_cli_gpu.py -x -q > gpurun_out/ryser11.txt 2>&1
./tests/cpp/test_permanent_device > gpurun_out/cpp11.txt 2>&1; echo "cpp rc=$?" >> gpurun_out/cpp11.txt
python - >> gpurun_out/ryser11.txt 2>&1 <<'PY'
import sys, time; sys.path.insert(0, '.')
import numpy as np, paper_1802_02779_b200 as pl
for n in (20, 22, 24):
    a = np.random.default_rng(n).uniform(-1, 1, (n, n))
    pl.ryser_permanent(a)
    t = time.perf_counter(); pl.ryser_permanent(a); dt = time.perf_counter() - t
    c = np.random.default_rng(n).standard_normal((n, n)) + 1j
    t2 = time.perf_counter(); pl.ryser_permanent(c); dt2 = time.perf_counter() - t2
    i = np.random.default_rng(n).integers(0, 2, (n, n))
    t3 = time.perf_counter(); pl.ryser_permanent(i); dt3 = time.perf_counter() - t3
    print(f"ryser n={n}: f64 {dt*1e3:.1f} ms, c128 {dt2*1e3:.1f} ms, i64 {dt3*1e3:.1f} ms")
PY
