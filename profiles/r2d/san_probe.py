"""Small exercise of the round-2d kernels (written for compute-sanitizer, which is closed on this pool; it runs as a plain self-check):
residue passes (small-order kernel, layer kernels on RModP), Ryser residue sums, overlapped
batch launches with PL_FLAG_INPUT_READY, the boson kernel with the flag."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1802_02779_b200 as pl  # noqa: E402
from paper_1802_02779_b200 import boson as B  # noqa: E402

assert pl.store_zechin_permanent(np.full((9, 9), 10 ** 6, dtype=np.int64)).value == 10 ** 54 * math.factorial(9)
assert pl.store_zechin_permanent(np.ones((21, 21), dtype=np.int64)).value == math.factorial(21)
assert pl.ryser_permanent(np.full((12, 12), 10 ** 9, dtype=np.int64)).value == 10 ** 108 * math.factorial(12)
rng = np.random.default_rng(1)
for dtype, n in ((np.int64, 5), (np.complex128, 5), (np.int64, 12)):
    count = 32 * 9 + 7
    a = rng.integers(0, 2, (count, n, n)).astype(dtype)
    want = pl.store_zechin_permanent_batch(a)
    bufs = [torch.from_numpy(a).cuda() for _ in range(2)]
    outs = [torch.zeros(count, dtype=bufs[0].dtype, device="cuda") for _ in range(2)]
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for i in range(6):
        pl.store_zechin_permanent_batch(bufs[i % 2], out=outs[i % 2], status=st, input_ready=True)
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy(), want)
itf = B.haar_unitary(10, 2)
host = B.distribution_probabilities(itf, [0, 1, 2])
out = torch.zeros(host.shape[0], dtype=torch.float64, device="cuda")
st = torch.zeros(1, dtype=torch.int32, device="cuda")
for _ in range(3):
    B.distribution_probabilities(itf, [0, 1, 2], out=out, status=st, input_ready=True)
torch.cuda.synchronize()
assert np.array_equal(out.cpu().numpy(), host)
print("san probe ok")
