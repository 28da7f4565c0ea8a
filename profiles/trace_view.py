"""Summarise a PL_WS_TRACE dump (CTA 0 event trace of one layer-kernel launch)."""
import sys
import numpy as np
cap = 65536
a = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(4, cap, 2)
names = {1: "slot-wait", 3: "stage-wait", 6: "empty-wait", 8: "slot-free-wait"}
t0 = min(int(a[r, 0, 0]) for r in range(4) if a[r, 0, 0])
for r, role in enumerate(["consumer g0", "consumer g1", "streamer g0", "publisher"]):
    n = int((a[r, :, 0] != 0).sum())
    if n == 0:
        continue
    t = a[r, :n, 0].astype(np.int64) - t0
    e = (a[r, :n, 1] & 0xff).astype(int)
    span = t[-1] - t[0]
    waits = {}
    for i in range(n - 1):
        if e[i] in names and e[i + 1] == e[i] + 1:
            waits.setdefault(names[e[i]], []).append(t[i + 1] - t[i])
    s = ", ".join(f"{k}: n={len(v)} total={sum(v) / span * 100:.1f}% mean={np.mean(v):.0f}cyc" for k, v in waits.items())
    print(f"{role:12s} events {n:6d} span {span / 1e3:.1f} kcyc  {s}")
