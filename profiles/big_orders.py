import sys, time
sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
for n in (33, 34):
    for dt in ("f", "c"):
        a = configs.uniform((n, n), seed=n) * 0.3
        if dt == "c":
            a = a + 1j * configs.uniform((n, n), seed=n + 1) * 0.3
        t0 = time.time(); v1 = pl.store_zechin_permanent(a).value; t1 = time.time()
        v2 = pl.store_zechin_permanent(a).value; t2 = time.time()
        print(n, dt, v1, v1 == v2, f"first {t1-t0:.2f}s second {t2-t1:.2f}s", flush=True)
