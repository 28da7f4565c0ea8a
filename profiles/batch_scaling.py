"""Kernel throughput of the batched n=5 path vs batch size (device-resident, event-timed, L2 flushed)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
big = torch.empty(2, 64 * 1024 * 1024, device="cuda")
for dt in ("c128", "i64"):
    for count in (25_000, 100_000, 400_000, 1_600_000):
        if dt == "c128":
            a = configs.uniform((count, 5, 5), seed=1) + 1j * configs.uniform((count, 5, 5), seed=2)
        else:
            a = configs.int_matrices(5, count, seed=3)
        t = torch.from_numpy(a).cuda()
        out = torch.empty(count, dtype=t.dtype, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        for _ in range(3):
            pl.store_zechin_permanent_batch(t, out=out, status=st)
        ts = []
        for _ in range(10):
            big[0].add_(1); big[1].sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); pl.store_zechin_permanent_batch(t, out=out, status=st); e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        us = sorted(x.elapsed_time(y) * 1000 for x, y in ts)[5]
        gbs = count * t[0].numel() * t.element_size() / us / 1e3
        print(f"{dt} {count:8d}: {us:8.1f} us  {count / us / 1e3:6.2f} G perm/s  {gbs:6.0f} GB/s")
