cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_ryser_gpu.py -x -q > gpurun_out/ry23.txt 2>&1
python - >> gpurun_out/ry23.txt 2>&1 <<'PY'
import sys, time; sys.path.insert(0, '.')
import numpy as np, paper_1802_02779_b200 as pl
for n in (20, 22, 24):
    a = np.random.default_rng(n).uniform(-1, 1, (n, n)); pl.ryser_permanent(a)
    t = time.perf_counter(); pl.ryser_permanent(a); dt = time.perf_counter() - t
    c = a + 1j * a; pl.ryser_permanent(c)
    t2 = time.perf_counter(); pl.ryser_permanent(c); dt2 = time.perf_counter() - t2
    print(f"ryser n={n}: f64 {dt*1e3:.1f} ms ({dt/2**n*1e9:.2f} ns/term), c128 {dt2*1e3:.1f} ms")
PY
