"""C3 (10k x 12x12 int64) and n = 10, 11 batches: parity against the oracle / golden SHA and timing,
for the current environment (PL_BATCH_F32_BLK=0 selects the subset-per-thread pack kernel)."""
import hashlib, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np, torch
import paper_1802_02779_b200 as pl
from oracle import oracle as O
from paper_1802_02779_b200 import configs

g = json.loads((Path(__file__).resolve().parents[2] / "tests/golden/goldens.json").read_text())
a = configs.c3()
out = pl.store_zechin_permanent_batch(a)
print("c3 sha ok", hashlib.sha256(np.ascontiguousarray(out).tobytes()).hexdigest() == g["c3"]["output_sha256"], flush=True)
print("c3 first 512 vs oracle", np.array_equal(out[:512], O.sz_batch(a[:512])))
for n in (10, 11, 12):
    for lo, hi in ((0, 2), (-1, 2), (-3, 4)):
        b = configs.int_matrices(n, 203, seed=77 + n, lo=lo, hi=hi)
        print("n", n, (lo, hi), np.array_equal(pl.store_zechin_permanent_batch(b), O.sz_batch(b)), flush=True)
ad = torch.from_numpy(a).cuda()
copies = [ad.clone() for _ in range(24)]  # 24 x 11.5 MB > L2
for c in copies[:3]:
    pl.store_zechin_permanent_batch(c)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for r in range(96):
    o = pl.store_zechin_permanent_batch(copies[r % 24])
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 96
print("c3 %.1f us per batch, %.1f M perm/s" % (ms * 1e3, 10000 / ms / 1e3))
