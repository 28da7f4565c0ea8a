"""Determinism probe of the layer kernel: every layer of one matrix is computed
once into `cur`, then recomputed R times from the same `prev` into `chk`; any
bitwise difference is reported with the ranks decoded into (tile F, offset).
Usage: python profiles/determinism_probe.py [n] [dtype c|f|c5] [R]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import math
import numpy as np
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
from paper_1802_02779_b200.sharded import device_hooks

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
dt = sys.argv[2] if len(sys.argv) > 2 else "c5"
R = int(sys.argv[3]) if len(sys.argv) > 3 else 3
if dt == "c5":
    a = torch.from_numpy(configs.c5()).cuda()
elif dt == "c":
    a = torch.from_numpy(configs.complex_uniform((n, n), seed=n)).cuda()
else:
    a = torch.from_numpy(configs.uniform((n, n), seed=n)).cuda()
layer_fn, top_fn = device_hooks(a)
L = max(math.comb(n, k) for k in range(2, n))
mk = lambda: torch.zeros(L + 8, dtype=a.dtype, device="cuda")
prev, cur, chk = mk(), mk(), mk()
D = 14
bad_total = 0
for k in range(2, n):
    ck = math.comb(n, k)
    layer_fn(k, prev, cur, 0, ck)
    if k >= 3:
        for r in range(R):
            chk.fill_(float("nan"))
            layer_fn(k, prev, chk, 0, ck)
            torch.cuda.synchronize()
            x = cur[:ck].view(torch.float64) if a.is_complex() else cur[:ck]
            y = chk[:ck].view(torch.float64) if a.is_complex() else chk[:ck]
            ne = (x.view(torch.int64) != y.view(torch.int64))
            if a.is_complex():
                ne = ne.view(-1, 2).any(dim=1)
            nbad = int(ne.sum().item())
            if nbad:
                bad_total += nbad
                idx = torch.nonzero(ne).flatten()[:12].cpu().tolist()
                info = []
                for q in idx:
                    mask = pl.colex_unrank(k, q)
                    F = mask >> D
                    m = k - bin(F).count("1")
                    base = 0
                    l = 1
                    ff = F
                    while ff:
                        h = (ff & -ff).bit_length() - 1
                        base += math.comb(D + h, m + l)
                        l += 1
                        ff &= ff - 1
                    info.append((q, hex(F), m, q - base))
                print(f"k={k} rep={r}: {nbad} mismatches; first (rank, F, m, offset): {info}", flush=True)
    prev, cur = cur, prev
    print(f"layer {k} done", flush=True)
print("value", top_fn(a, prev), "total mismatches", bad_total)
