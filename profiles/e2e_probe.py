"""Time the pieces of the host-buffer (e2e) path for one config."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
a = configs.generate(name)
a_host = torch.from_numpy(a).pin_memory()
out_host = torch.empty(a.shape[0], dtype=a_host.dtype).pin_memory()
st = torch.cuda.current_stream()
for i in range(4):
    torch.cuda.synchronize(); t = time.perf_counter()
    pl.store_zechin_permanent_batch(a_host, out=out_host, stream=st)
    torch.cuda.synchronize(); print(f"{name} host-path call {i}: {1000*(time.perf_counter()-t):.3f} ms")
t = time.perf_counter(); d = a_host.cuda(non_blocking=True); torch.cuda.synchronize(); print(f"H2D alone {1000*(time.perf_counter()-t):.3f} ms")
o = torch.empty(a.shape[0], dtype=d.dtype, device="cuda"); s = torch.zeros(1, dtype=torch.int32, device="cuda")
for i in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    pl.store_zechin_permanent_batch(d, out=o, status=s)
    torch.cuda.synchronize(); print(f"device call {i}: {1000*(time.perf_counter()-t):.3f} ms")
