"""Quick device timing of configs through the public API (device-resident inputs)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["c4", "c5"]
fma = "--fma" in sys.argv
for name in names:
    a = torch.from_numpy(configs.generate(name)).cuda()
    out = torch.empty(a.shape[0], dtype=a.dtype, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    reps = 3 if name in ("c5",) else 10
    for _ in range(2):
        pl.store_zechin_permanent_batch(a, out=out, status=st, fma=fma)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); pl.store_zechin_permanent_batch(a, out=out, status=st, fma=fma); e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    ms = [x.elapsed_time(y) for x, y in ts]
    print(f"{name} fma={fma}: min {min(ms):.3f} ms  median {sorted(ms)[len(ms)//2]:.3f} ms  value {out[0].item()}")
