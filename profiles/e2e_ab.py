"""e2e of the host-pointer batch call (bench.py's e2e loop), for the chunked
upload/compute/download pipeline vs one upload + kernel + download
(PL_HOST_PIPE=0), alternating in one process is not possible (read once), so
run twice."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
tag = os.environ.get("PL_HOST_PIPE", "1")
for name in ("c2", "c1", "c3"):
    a = torch.from_numpy(configs.generate(name)).pin_memory()
    out = torch.empty(a.shape[0], dtype=a.dtype).pin_memory()
    st = torch.cuda.current_stream()
    for _ in range(5):
        pl.store_zechin_permanent_batch(a, out=out, stream=st)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        pl.store_zechin_permanent_batch(a, out=out, stream=st)
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    print(f"pipe={tag} {name}: median {ts[10] * 1000:.0f} us  min {ts[0] * 1000:.0f} us  "
          f"{a.shape[0] / (ts[10] / 1000) / 1e6:.1f} M/s")
