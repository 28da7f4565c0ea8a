"""Nondeterminism vs buffer reuse: the layer chain of one matrix through
pl_sz_layer with B rotating layer buffers (B = 2 is the library's ping-pong),
repeated R times; prints each value and the number of distinct values.
Usage: python profiles/rotation_probe.py n B R"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import math
import torch
from paper_1802_02779_b200 import configs
from paper_1802_02779_b200.sharded import device_hooks

n, B, R = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
a = torch.from_numpy(configs.uniform((n, n), seed=n) * 0.3 + 1j * configs.uniform((n, n), seed=n + 1) * 0.3).cuda()
layer_fn, top_fn = device_hooks(a)
L = max(math.comb(n, k) for k in range(2, n)) + 16
bufs = [torch.zeros(L, dtype=a.dtype, device="cuda") for _ in range(B)]
vals = []
for r in range(R):
    for k in range(2, n):
        layer_fn(k, bufs[(k - 1) % B], bufs[k % B], 0, math.comb(n, k))
    v = complex(top_fn(a, bufs[(n - 1) % B]))
    vals.append(v)
    print(n, B, r, v.real.hex(), v.imag.hex(), flush=True)
print(f"n={n} B={B}: distinct values {len(set(vals))} of {R}")
