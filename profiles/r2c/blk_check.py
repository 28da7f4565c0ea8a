"""Register-blocked engine (sz_blk.cuh): bitwise check against the oracle and timing of C4 / C5."""
import json, sys, time
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1802_02779_b200 as pl
from oracle import oracle as O
from paper_1802_02779_b200 import configs

def hexf(x):
    return float(x).hex()

bad = 0
for n in list(range(15, 25)):
    a = configs.uniform((n, n), seed=3000 + n)
    got = pl.store_zechin_permanent(a).value
    want = O.sz_f64(a)
    ok = hexf(got) == hexf(want)
    bad += not ok
    print("f64", n, ok, got, want, flush=True)
for n in list(range(15, 23)):
    a = configs.complex_uniform((n, n), seed=2000 + n)
    got = complex(pl.store_zechin_permanent(a).value)
    want = complex(O.sz_batch(a[None])[0])
    ok = (hexf(got.real), hexf(got.imag)) == (hexf(want.real), hexf(want.imag))
    bad += not ok
    print("c128", n, ok, got, want, flush=True)
g = json.loads((Path(__file__).resolve().parents[2] / "tests/golden/goldens.json").read_text())
import torch
def timeit(a, reps, fma=False):
    pl.store_zechin_permanent(a, fma=fma)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        v = pl.store_zechin_permanent(a, fma=fma).value
    torch.cuda.synchronize()
    return v, (time.perf_counter() - t0) / reps * 1e3
a = configs.c4()
v, ms = timeit(a, 20)
print("C4", hexf(v) == g["c4"]["value_hex"], v, "%.3f ms" % ms, flush=True)
bad += hexf(v) != g["c4"]["value_hex"]
v, ms = timeit(a, 20, fma=True)
print("C4 fma", v, "%.3f ms" % ms, flush=True)
a = configs.c5()
v, ms = timeit(a, 3)
v = complex(v)
ok = [hexf(v.real), hexf(v.imag)] == g["c5"]["value_hex"]
bad += not ok
print("C5", ok, v, "%.2f ms" % ms, flush=True)
v, ms = timeit(a, 3, fma=True)
print("C5 fma", v, "%.2f ms" % ms, flush=True)
print("BAD", bad)
