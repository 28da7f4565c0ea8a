"""A/B of the n <= 5 batch kernels (PL_BATCH_KERNEL=warp|pipe set by the caller):
event-timed single calls after an L2 flush, C1/C2 and batch-size scaling."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
big = torch.empty(2, 64 * 1024 * 1024, device="cuda")
kind = os.environ.get("PL_BATCH_KERNEL", "pipe")


def timed(a, reps=30):
    out = torch.empty(a.shape[0], dtype=a.dtype, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for _ in range(5):
        pl.store_zechin_permanent_batch(a, out=out, status=st)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        big[0].add_(1); big[1].sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); pl.store_zechin_permanent_batch(a, out=out, status=st); e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    s = sorted(x.elapsed_time(y) * 1000 for x, y in ts)
    return s[len(s) // 2], out


for name in ("c1", "c2"):
    a_np = configs.generate(name)
    a = torch.from_numpy(a_np).cuda()
    us, out = timed(a)
    print(f"{kind} {name}: median {us:.2f} us  {a.shape[0] / us / 1e3:.2f} G perm/s  sha {configs.sha256(out.cpu().numpy())[:16]}")
for count in (25_000, 400_000, 1_600_000):
    a = torch.from_numpy(configs.uniform((count, 5, 5), seed=1) + 1j * configs.uniform((count, 5, 5), seed=2)).cuda()
    us, _ = timed(a, 10)
    print(f"{kind} c128 {count}: {us:.1f} us  {count * 400 / us / 1e3:.0f} GB/s")
