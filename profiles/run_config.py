"""Run one config once through the public API (for ncu / sanitizer captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_1802_02779_b200 as pl  # noqa: E402
from paper_1802_02779_b200 import configs  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
fma = "--fma" in sys.argv
a = torch.from_numpy(configs.generate(name)).cuda()
out = pl.store_zechin_permanent_batch(a, fma=fma)
torch.cuda.synchronize()
print(name, out[:4].cpu().numpy())
