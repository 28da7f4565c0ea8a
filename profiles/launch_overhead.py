"""Event-timed C1/C2 batched calls: single calls bracketed by events vs. back-to-back runs."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
for name in (sys.argv[1:] or ["c2", "c1"]):
    a = torch.from_numpy(configs.generate(name)).cuda()
    out = torch.empty(a.shape[0], dtype=a.dtype, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(5):
        pl.store_zechin_permanent_batch(a, out=out, status=st, stream=stream)
    torch.cuda.synchronize()
    big = torch.empty(2, 64 * 1024 * 1024, device="cuda")
    single = []
    for _ in range(20):
        big[0].add_(1); big[1].sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); pl.store_zechin_permanent_batch(a, out=out, status=st, stream=stream); e1.record(stream)
        single.append((e0, e1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(50):
        pl.store_zechin_permanent_batch(a, out=out, status=st, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    s = sorted(x.elapsed_time(y) * 1000 for x, y in single)
    print(f"{name}: single (flushed) median {s[len(s)//2]:.2f} us, min {s[0]:.2f}; back-to-back {e0.elapsed_time(e1) * 1000 / 50:.2f} us/call")
