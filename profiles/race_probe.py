"""Localise nondeterminism in the layer DP: run the whole chain of layers
back to back (as a normal permanent call does, programmatic dependent launch
between layers) R times, every layer into its own buffer, then compare the
runs layer by layer. The first layer where runs disagree is where the bad
entries arose; their ranks are decoded into (tile F, m, offset in tile).
Usage: python profiles/race_probe.py [n] [R] [rounds]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import math
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
from paper_1802_02779_b200.sharded import device_hooks

n = int(sys.argv[1]) if len(sys.argv) > 1 else 31
R = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rounds = int(sys.argv[3]) if len(sys.argv) > 3 else 2
D = 14
a = torch.from_numpy(configs.complex_uniform((n, n), seed=n) * 0.3).cuda()
layer_fn, top_fn = device_hooks(a)
offs, tot = {}, 0
for k in range(2, n):
    offs[k] = tot
    tot += (math.comb(n, k) + 16 + 15) // 16 * 16
bufs = [torch.zeros(tot, dtype=a.dtype, device="cuda") for _ in range(R)]
lay = lambda b, k: bufs[b][offs[k]:offs[k] + math.comb(n, k)]


def decode(k, q):
    mask = pl.colex_unrank(k, q)
    F = mask >> D
    m = k - bin(F).count("1")
    base, l, ff = 0, 1, F
    while ff:
        h = (ff & -ff).bit_length() - 1
        base += math.comb(D + h, m + l)
        l += 1
        ff &= ff - 1
    return (q, hex(F), m, q - base)


for rd in range(rounds):
    for b in range(R):
        bufs[b].fill_(float("nan"))
    torch.cuda.synchronize()
    vals = []
    for b in range(R):
        for k in range(2, n):
            layer_fn(k, lay(b, k - 1) if k > 2 else lay(b, 2), lay(b, k), 0, math.comb(n, k))
        vals.append(top_fn(a, lay(b, n - 1)))
    torch.cuda.synchronize()
    print(f"round {rd}: values {[complex(v) for v in vals]}", flush=True)
    for k in range(2, n):
        ref = lay(0, k).view(torch.int64).view(-1, 2)
        for b in range(1, R):
            ne = (lay(b, k).view(torch.int64).view(-1, 2) != ref).any(dim=1)
            c = int(ne.sum().item())
            if c:
                idx = torch.nonzero(ne).flatten()[:10].cpu().tolist()
                nan0 = int(torch.isnan(lay(0, k).view(torch.float64)).sum().item())
                nanb = int(torch.isnan(lay(b, k).view(torch.float64)).sum().item())
                print(f"  layer {k}: run {b} vs 0: {c} entries differ (NaNs run0 {nan0}, run{b} {nanb}); "
                      f"first {[decode(k, q) for q in idx]}", flush=True)
        # only report the first differing layer per round in detail
print("done")
