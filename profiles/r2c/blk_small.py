"""Small orders through the block engine with the current environment (debug of multi-tile CTAs)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import paper_1802_02779_b200 as pl
from oracle import oracle as O
from paper_1802_02779_b200 import configs
for n in [int(x) for x in sys.argv[1:]] or [16, 17, 18]:
    a = configs.uniform((n, n), seed=3000 + n)
    got = pl.store_zechin_permanent(a).value
    print("f64", n, float(got).hex() == float(O.sz_f64(a)).hex(), flush=True)
    c = configs.complex_uniform((n, n), seed=2000 + n)
    v = complex(pl.store_zechin_permanent(c).value); w = complex(O.sz_batch(c[None])[0])
    print("c128", n, v == w, flush=True)
