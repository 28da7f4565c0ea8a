"""H2D of 40 MB pinned: one copy, chunked on one stream, chunked on 2/4 streams (copy engines)."""
import torch
torch.cuda.init()
a = torch.empty(40_000_000 // 8, dtype=torch.float64).pin_memory(); a.fill_(1.0)
d = torch.empty(a.shape, dtype=a.dtype, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]

def run(nstreams, chunk_mb):
    ch = chunk_mb * 1024 * 1024 // 8
    main = torch.cuda.current_stream()
    for s in streams[:nstreams]:
        s.wait_stream(main)
    for i, off in enumerate(range(0, a.numel(), ch)):
        s = streams[i % nstreams]
        with torch.cuda.stream(s):
            d[off:off + ch].copy_(a[off:off + ch], non_blocking=True)
    for s in streams[:nstreams]:
        main.wait_stream(s)

out = []
for ns, cm in ((1, 40), (1, 8), (1, 2), (2, 8), (2, 2), (4, 2), (4, 1)):
    for _ in range(3):
        run(ns, cm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        run(ns, cm)
    e1.record(); torch.cuda.synchronize()
    out.append(f"{ns}s/{cm}MB {10 * 40e6 / (e0.elapsed_time(e1) / 1e3) / 1e9:.1f}")
print("H2D GB/s:", ", ".join(out))
