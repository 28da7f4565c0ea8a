"""complex128 batches of 6 <= n <= 13 (boson outcomes with 7-13 photons take this path):
event-timed after an L2 flush, with the oracle check."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
from oracle import oracle as O
big = torch.empty(2, 64 * 1024 * 1024, device="cuda")
tag = os.environ.get("TAG", "")
for n, count in ((7, 20000), (10, 10000), (12, 5000)):
    a_np = configs.complex_uniform((count, n, n), seed=n)
    a = torch.from_numpy(a_np).cuda()
    out = torch.empty(count, dtype=a.dtype, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(3):
        pl.store_zechin_permanent_batch(a, out=out, status=st)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        big[0].add_(1); big[1].sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); pl.store_zechin_permanent_batch(a, out=out, status=st); e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    us = sorted(x.elapsed_time(y) * 1000 for x, y in ts)[5]
    ok = np.array_equal(out.cpu().numpy().view(np.uint64), O.sz_batch(a_np).view(np.uint64))
    print(f"{tag} c128 n={n} x{count}: {us:.1f} us  {count / us:.3f} M perm/s  bitwise {ok}", flush=True)
