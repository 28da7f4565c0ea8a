"""C3 (10k x 12x12 int64) and other 6 <= n <= 12 batches: event-timed after an L2 flush, with the oracle check."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os
import numpy as np
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
from oracle import oracle as O
big = torch.empty(2, 64 * 1024 * 1024, device="cuda")
tag = os.environ.get("TAG", "")
cases = [("c3", configs.c3()), ("i64 n=8 x50k", configs.int_matrices(8, 50_000, seed=8)),
         ("f64 n=10 x20k", configs.uniform((20_000, 10, 10), seed=10)), ("i64 big n=12", configs.int_matrices(12, 4000, seed=5, lo=-10, hi=10))]
for name, a_np in cases:
    a = torch.from_numpy(a_np).cuda()
    out = torch.empty(a.shape[0], dtype=a.dtype, device="cuda")
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
    ok = np.array_equal(out.cpu().numpy(), O.sz_batch(a_np)) if a_np.dtype != np.float64 else \
        bool(np.max(np.abs(out.cpu().numpy() - O.sz_batch(a_np)) / np.abs(O.sz_batch(a_np))) < 1e-9)
    print(f"{tag} {name}: {us:.1f} us  {a.shape[0] / us:.3f} M perm/s  status {int(st.item())}  ok {ok}", flush=True)
