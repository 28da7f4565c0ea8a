import sys; sys.path.insert(0, ".")
import numpy as np
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
n = 34
a = configs.uniform((n, n), seed=n) * 0.3 + 1j * configs.uniform((n, n), seed=n + 1) * 0.3
c = a[:, ::-1].copy()
for rep in range(3):
    pa = complex(pl.store_zechin_permanent(a).value)
    pc = complex(pl.store_zechin_permanent(c).value)
    print(rep, pa, pc, abs(pc - pa) / abs(pa), flush=True)
a5 = configs.c5()
for rep in range(4):
    print("c5", complex(pl.store_zechin_permanent(a5).value), flush=True)
