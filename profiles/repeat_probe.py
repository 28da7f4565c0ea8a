"""Repeat one large permanent R times and print each value (nondeterminism check).
Usage: python profiles/repeat_probe.py [c5|n34] [R]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
which = sys.argv[1] if len(sys.argv) > 1 else "c5"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 6
if which == "c5":
    a = configs.c5()
else:
    n = int(which[1:])
    a = configs.uniform((n, n), seed=n) * 0.3 + 1j * configs.uniform((n, n), seed=n + 1) * 0.3
vals = [complex(pl.store_zechin_permanent(a).value) for _ in range(R)]
for v in vals:
    print(which, v.real.hex(), v.imag.hex(), flush=True)
print(which, "distinct values:", len(set(vals)))
