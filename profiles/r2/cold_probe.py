"""Split a cold C5 call: module load + tables (a small n = 20 complex call
first), then the C5-specific first call (schedules, 19 GB scratch), then a
warm call."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
torch.cuda.init(); torch.zeros(1, device="cuda"); torch.cuda.synchronize()
from paper_1802_02779_b200 import configs
c5 = configs.generate("c5")
small = configs.complex_uniform((1, 20, 20), seed=3)
t0 = time.perf_counter()
import paper_1802_02779_b200 as pl
t1 = time.perf_counter(); pl.store_zechin_permanent_batch(small)
t2 = time.perf_counter(); pl.store_zechin_permanent_batch(small)
t3 = time.perf_counter(); pl.store_zechin_permanent_batch(c5)
t4 = time.perf_counter(); pl.store_zechin_permanent_batch(c5)
t5 = time.perf_counter()
print(f"import {1e3*(t1-t0):.1f} ms; first n=20 call {1e3*(t2-t1):.1f}; second n=20 {1e3*(t3-t2):.1f}; "
      f"first C5 {1e3*(t4-t3):.1f}; second C5 {1e3*(t5-t4):.1f}")
