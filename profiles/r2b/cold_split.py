"""Cold-call split: a tiny call first (module load), then the first C4 call."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
torch.cuda.init(); torch.zeros(1, device="cuda"); torch.cuda.synchronize()
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
c4 = configs.generate("c4")
t0 = time.perf_counter(); pl.store_zechin_permanent(np.eye(3))
t1 = time.perf_counter(); pl.store_zechin_permanent(np.eye(3))
t2 = time.perf_counter(); pl.store_zechin_permanent_batch(configs.uniform((1, 16, 16), seed=1))
t3 = time.perf_counter(); pl.store_zechin_permanent_batch(c4)
t4 = time.perf_counter(); pl.store_zechin_permanent_batch(c4)
t5 = time.perf_counter()
print(f"first tiny {1e3*(t1-t0):.1f} ms; second tiny {1e3*(t2-t1):.1f}; first n=16 {1e3*(t3-t2):.1f}; "
      f"first C4 {1e3*(t4-t3):.1f}; second C4 {1e3*(t5-t4):.1f}", flush=True)
