"""Time C4 / C5 (device-resident input, events) with the current environment's engine settings."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs

def timeit(name, reps):
    a = torch.from_numpy(configs.generate(name)).cuda()
    for _ in range(2):
        out = pl.store_zechin_permanent_batch(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = pl.store_zechin_permanent_batch(a)
    e1.record()
    torch.cuda.synchronize()
    print(name, out.cpu().numpy(), "%.4f ms" % (e0.elapsed_time(e1) / reps), flush=True)

for name in sys.argv[1:] or ["c4", "c5"]:
    timeit(name, 20 if name == "c4" else 3)
