"""Where does the C2 step time go? Event pairs around (a) an empty kernel after
the L2 flush, (b) the batch kernel after the flush, (c) the batch kernel back
to back, (d) the batch kernel after the flush with an empty kernel between."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs

a = torch.from_numpy(configs.generate("c2")).cuda()
out = torch.empty(a.shape[0], dtype=a.dtype, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
stream = torch.cuda.current_stream()
big = torch.empty(2, 64 * 1024 * 1024, device="cuda")
call = lambda: pl.store_zechin_permanent_batch(a, out=out, status=st, stream=stream)
for _ in range(5):
    call()
torch.cuda.synchronize()


def timed(body, flush=True, reps=30):
    ts = []
    for _ in range(reps):
        if flush:
            big[0].add_(1); big[1].sum()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); body(); e1.record(stream)
        ts.append((e0, e1))
    torch.cuda.synchronize()
    s = sorted(x.elapsed_time(y) * 1000 for x, y in ts)
    return s[len(s) // 2], s[0]


print("empty (sleep 0) after flush: med %.2f min %.2f us" % timed(lambda: torch.cuda._sleep(0)))
print("nothing after flush:         med %.2f min %.2f us" % timed(lambda: None))
print("batch after flush:           med %.2f min %.2f us" % timed(call))
print("batch after flush+sleep0:    med %.2f min %.2f us" % timed(lambda: (torch.cuda._sleep(0), call())))
print("batch no flush:              med %.2f min %.2f us" % timed(call, flush=False))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(100):
    call()
e1.record(stream)
torch.cuda.synchronize()
print("back-to-back: %.2f us/call" % (e0.elapsed_time(e1) * 10))
