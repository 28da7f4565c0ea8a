"""Pinned host -> device bandwidth for a 40 MB batch: one copy vs split across streams."""
import torch
n = 40_000_000
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
for parts in (1, 2, 4):
    for _ in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        chunk = n // parts
        for i in range(parts):
            s = streams[i]
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for i in range(parts):
            torch.cuda.current_stream().wait_stream(streams[i])
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{parts} stream(s): {ms * 1000:.0f} us, {n / ms / 1e6:.1f} GB/s")
hd = torch.empty(1_600_000, dtype=torch.uint8).pin_memory()
dd = torch.empty(1_600_000, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); hd.copy_(dd, non_blocking=True); e1.record(); torch.cuda.synchronize()
print(f"D2H 1.6 MB: {e0.elapsed_time(e1) * 1000:.0f} us")
