"""Exact big-integer path (csrc/bigint.cu): wall time of the public call per order, against the
int64 attempt alone; run under ncu for the launch list (profiles/r2d/bigint_launches.md)."""
import math
import sys
import time

import numpy as np

sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[2]))

import paper_1802_02779_b200 as pl

orders = [int(v) for v in sys.argv[1:]] or [10, 14, 21, 24, 26, 30, 32]
for n in orders:
    a = np.ones((n, n), dtype=np.int64) * (3 if n < 21 else 1)
    a[0, 0] = 10 ** 12 if n < 21 else 1  # leave int64 at small orders too
    want = None
    ts = []
    for _ in range(4):
        t0 = time.perf_counter()
        v = pl.store_zechin_permanent(a).value
        ts.append(time.perf_counter() - t0)
    if n >= 21:
        assert v == math.factorial(n), (n, v)
    bits = sum(int(np.abs(r).sum()).bit_length() for r in a)
    print(f"n={n} passes={max(1, (bits + 31) // 30)} result_bits={v.bit_length()} "
          f"first={1e3 * ts[0]:.2f} ms steady={1e3 * min(ts[1:]):.2f} ms", flush=True)
