"""Localise a nondeterministic layer: run the layer chain back to back
(programmatic dependent launch between layers) with every layer archived in
its own buffer, then recompute each layer alone (synchronised) from the
archived previous layer and compare bitwise. Mismatching ranks are decoded
into (tile F, m, offset in tile, chunk).
Usage: python profiles/archive_probe.py n rounds"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import math
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
from paper_1802_02779_b200.sharded import device_hooks

n, rounds = int(sys.argv[1]), int(sys.argv[2])
D = 14
a = torch.from_numpy(configs.uniform((n, n), seed=n) * 0.3 + 1j * configs.uniform((n, n), seed=n + 1) * 0.3).cuda()
layer_fn, top_fn = device_hooks(a)
offs, tot = {}, 0
for k in range(2, n):
    offs[k] = tot
    tot += (math.comb(n, k) + 16 + 15) // 16 * 16
arch = torch.empty(tot, dtype=a.dtype, device="cuda")
scratch = torch.empty(max(math.comb(n, k) for k in range(2, n)) + 16, dtype=a.dtype, device="cuda")
lay = lambda k: arch[offs[k]:offs[k] + math.comb(n, k)]


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
    return (q, hex(F), m, q - base, (q - base) // 256)


for rd in range(rounds):
    arch.view(torch.float64).fill_(float("nan"))
    torch.cuda.synchronize()
    for k in range(2, n):
        layer_fn(k, lay(k - 1) if k > 2 else lay(2), lay(k), 0, math.comb(n, k))
    v = complex(top_fn(a, lay(n - 1)))
    bad = 0
    for k in range(3, n):
        ck = math.comb(n, k)
        layer_fn(k, lay(k - 1), scratch, 0, ck)
        torch.cuda.synchronize()
        ne = (scratch[:ck].view(torch.int64).view(-1, 2) != lay(k).view(torch.int64).view(-1, 2)).any(dim=1)
        c = int(ne.sum().item())
        if c:
            bad += c
            idx = torch.nonzero(ne).flatten()
            nan = int(torch.isnan(lay(k).view(torch.float64).view(-1, 2)[idx]).any(dim=1).sum().item())
            first = [decode(k, q) for q in idx[:16].cpu().tolist()]
            print(f"round {rd} layer {k}: {c} entries differ from a synchronised recompute "
                  f"({nan} of them NaN in the chained run); first {first}", flush=True)
            print("  chained:", [complex(x) for x in lay(k)[idx[:4]].cpu().tolist()],
                  " recomputed:", [complex(x) for x in scratch[idx[:4]].cpu().tolist()], flush=True)
            break  # later layers inherit the error
    print(f"round {rd}: value {v}, bad entries {bad}", flush=True)
