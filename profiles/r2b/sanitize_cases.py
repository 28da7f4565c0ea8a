"""Small invocations of every round-2 kernel, for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
from paper_1802_02779_b200.sharded import device_hooks, device_overlap_hooks, top_block
from math import comb

rng = np.random.default_rng(0)
which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "f32"):
    a = configs.int_matrices(12, 37, seed=1, lo=0, hi=1); a[3] = 1
    print("f32 pack", pl.store_zechin_permanent_batch(a)[:3])
if which in ("all", "lean"):
    c = rng.standard_normal((17, 17)) + 1j * rng.standard_normal((17, 17))
    print("lean single", pl.store_zechin_permanent(c).value)
    b = rng.uniform(-1, 1, (3, 16, 16))
    print("lean batched", pl.store_zechin_permanent_batch(b)[:2])
    i = rng.integers(0, 2, (3, 16, 16)).astype(np.int64)
    print("lean batched int", pl.store_zechin_permanent_batch(i)[:2])
if which in ("all", "ws"):
    f = rng.uniform(-1, 1, (21, 21))
    print("ws", pl.store_zechin_permanent(f).value)
if which in ("all", "ryser"):
    print("ryser", pl.ryser_permanent(rng.uniform(-1, 1, (10, 10))).value,
          pl.ryser_permanent(rng.integers(-3, 4, (9, 9))).value)
if which in ("all", "overlap"):
    n, world = 16, 4
    a = torch.from_numpy(rng.uniform(-1, 1, (n, n))).cuda()
    lf, tf = device_hooks(a)
    hooks = [device_overlap_hooks(a, lf, g, world) for g in range(world)]
    size = max(comb(n, k) for k in range(2, n)) + 64
    reps = [[torch.zeros(size, dtype=a.dtype, device="cuda") for _ in range(2)] for _ in range(world)]
    for k in range(2, n):
        for g in range(world):
            prev, cur = reps[g]
            r0, r1 = top_block(n, k, world, g)
            if r1 > r0:
                if k == 2:
                    lf(k, prev, cur, r0, r1)
                else:
                    hooks[g][0](k, prev, cur)
        if k >= 3:
            for g in range(world):
                for t in range(2):
                    if g >> t & 1:
                        h = g ^ (1 << t)
                        h0, h1 = top_block(n, k - 1, world, h)
                        reps[g][0][h0:h1] = reps[h][0][h0:h1]
            for g in range(world):
                r0, r1 = top_block(n, k, world, g)
                if r1 > r0:
                    hooks[g][1](k, reps[g][0], reps[g][1])
        for g in range(world):
            reps[g].reverse()
    torch.cuda.synchronize()
    print("overlap ok")
