"""H2D bandwidth of pinned buffers, several allocations per process (bimodal e2e investigation)."""
import torch, time
torch.cuda.init()
res = []
for trial in range(4):
    a = torch.empty(40_000_000 // 8, dtype=torch.float64).pin_memory()
    a.fill_(1.0)
    d = torch.empty(a.shape, dtype=a.dtype, device="cuda")
    for _ in range(3):
        d.copy_(a, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        d.copy_(a, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    res.append(20 * 40e6 / (e0.elapsed_time(e1) / 1e3) / 1e9)
print("H2D GB/s per pinned allocation:", [round(x, 1) for x in res], "is_pinned", a.is_pinned())
