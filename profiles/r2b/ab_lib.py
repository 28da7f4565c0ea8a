"""A/B timing of whole single-matrix runs through the C ABI of any library build.

    python profiles/r2b/ab_lib.py <lib.so> [c4 c5 ...] [--fma] [--reps N] [--graph]

Calls pl_sz_permanent_batch (count 1, device pointers) only, so it works with
older library builds; device-event timing after two warm-up calls.
"""
import ctypes
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch

from paper_1802_02779_b200 import configs

lib = ctypes.CDLL(sys.argv[1])
names = [a for a in sys.argv[2:] if a.startswith("c")] or ["c4", "c5"]
fma = "--fma" in sys.argv
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 0
lib.pl_sz_permanent_batch.restype = ctypes.c_int
lib.pl_last_error.restype = ctypes.c_char_p
DT = {np.int64: 0, np.float64: 1, np.complex128: 2}
for name in names:
    a_np = configs.generate(name)
    a = torch.from_numpy(a_np).cuda()
    out = torch.empty(a.shape[0], dtype=a.dtype, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    dt = DT[a_np.dtype.type]
    flags = 0x1 | 0x4 | (0x2 if fma else 0)
    stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)

    def call():
        rc = lib.pl_sz_permanent_batch(dt, a.shape[1], a.shape[0], ctypes.c_void_p(a.data_ptr()),
                                       ctypes.c_void_p(out.data_ptr()), flags, None, stream,
                                       ctypes.c_void_p(st.data_ptr()))
        assert rc == 0, lib.pl_last_error()

    for _ in range(2):
        call()
    torch.cuda.synchronize()
    if "--graph" in sys.argv:
        g = torch.cuda.CUDAGraph()
        s_ = torch.cuda.Stream()
        with torch.cuda.stream(s_):
            stream = ctypes.c_void_p(s_.cuda_stream)
            with torch.cuda.graph(g, stream=s_):
                call()
        torch.cuda.synchronize()
        call = g.replay  # noqa: F811
    ts = []
    for _ in range(reps or (3 if name == "c5" else 10)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        ts.append((e0, e1))
    torch.cuda.synchronize()
    import time as _t
    h0 = _t.perf_counter()
    for _ in range(5):
        call()
    h1 = _t.perf_counter()
    torch.cuda.synchronize()
    h2 = _t.perf_counter()
    print(f"  host enqueue {1e3 * (h1 - h0) / 5:.3f} ms/call, enqueue+drain {1e3 * (h2 - h0) / 5:.3f} ms/call")
    ms = sorted(x.elapsed_time(y) for x, y in ts)
    print(f"{Path(sys.argv[1]).name} {name} fma={fma}: min {ms[0]:.3f} ms median {ms[len(ms)//2]:.3f} ms "
          f"value {out[0].item()}", flush=True)
