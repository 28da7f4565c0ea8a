import sys; sys.path.insert(0, ".")
import numpy as np, torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
from oracle import oracle as O
for name in ("c2", "c1"):
    a = configs.generate(name)[:3000 + 7]
    out = pl.store_zechin_permanent_batch(torch.from_numpy(a).cuda()).cpu().numpy()
    print(name, np.array_equal(out, O.sz_batch(a)), flush=True)
