"""Cross-check of the e2e number: the C2 API call with pinned host buffers vs a bare pinned H2D copy."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import time
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
a = torch.from_numpy(configs.generate("c2")).pin_memory()
out = torch.empty(a.shape[0], dtype=a.dtype).pin_memory()
st = torch.cuda.current_stream()
for _ in range(3):
    pl.store_zechin_permanent_batch(a, out=out, stream=st)
torch.cuda.synchronize()
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record(st)
    pl.store_zechin_permanent_batch(a, out=out, stream=st)
    e1.record(st)
    e1.synchronize()
    wall = time.perf_counter() - t
    print(f"api call: events {e0.elapsed_time(e1) * 1000:.0f} us, wall {wall * 1e6:.0f} us, "
          f"{a.numel() * 16 / (wall * 1e9):.1f} GB/s by wall")
d = torch.empty_like(a, device="cuda")
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); d.copy_(a, non_blocking=True); e1.record(st); e1.synchronize()
    wall = time.perf_counter() - t
    print(f"bare H2D 40 MB: events {e0.elapsed_time(e1) * 1000:.0f} us, wall {wall * 1e6:.0f} us")
