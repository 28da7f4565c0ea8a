"""A/B of PL_FLAG_INPUT_READY on the shared-memory batch kernels (6 <= n <= 14): a CUDA graph of 40
back-to-back batch calls on rotating inputs, replayed between one event pair, with and without the flag."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1802_02779_b200 as pl  # noqa: E402

rng = np.random.default_rng(5)
for dtype, n, count in (("int64", 8, 50000), ("float64", 8, 50000), ("complex128", 8, 50000), ("complex128", 12, 10000)):
    if dtype == "int64":
        a = rng.integers(-3, 4, (count, n, n)).astype(np.int64)
    elif dtype == "float64":
        a = rng.uniform(-1, 1, (count, n, n))
    else:
        a = rng.uniform(-1, 1, (count, n, n)) + 1j * rng.uniform(-1, 1, (count, n, n))
    reps = max(3, -(-(320 << 20) // a.nbytes))
    bufs = [torch.from_numpy(a).cuda() for _ in range(reps)]
    out = torch.zeros(count, dtype=bufs[0].dtype, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    res = {}
    for ready in (False, True, False, True):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for i in range(2):
                pl.store_zechin_permanent_batch(bufs[i], out=out, status=st, stream=s, input_ready=ready)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for i in range(40):
                pl.store_zechin_permanent_batch(bufs[i % reps], out=out, status=st, stream=s, input_ready=ready)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(ready, []).append(e0.elapsed_time(e1) / 40 * 1e3)
    print(f"{dtype} n={n} count={count}: without {min(res[False]):.1f} us/step, with {min(res[True]):.1f} us/step", flush=True)
