"""One device-resident call per config (C1..C5), in one process: the ncu launch
list of round 2 (profiles/r2b/capture.sh)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import torch  # noqa: E402

import paper_1802_02779_b200 as pl  # noqa: E402
from paper_1802_02779_b200 import configs  # noqa: E402

names = sys.argv[1:] or ["c1", "c2", "c3", "c4", "c5"]
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MiB > L2
for name in names:
    a = torch.from_numpy(configs.generate(name)).cuda()
    for _ in range(2):  # second call is the warm one (tables, scratch cached)
        flush.zero_()  # inputs come from HBM, as in bench.py (rotating copies / L2 flush)
        out = pl.store_zechin_permanent_batch(a)
    torch.cuda.synchronize()
    print(name, out[:2].cpu().numpy(), flush=True)
