"""Split a cold C4 call (PL_COLD_LOG=1 prints the one-time builds)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import numpy as np
import torch
torch.cuda.init(); torch.zeros(1, device="cuda"); torch.cuda.synchronize()
t0 = time.perf_counter()
from paper_1802_02779_b200 import configs
ti = time.perf_counter()
c4 = configs.generate("c4")
import paper_1802_02779_b200 as pl
import ctypes
t1 = time.perf_counter(); pl.store_zechin_permanent_batch(c4)
t2 = time.perf_counter(); pl.store_zechin_permanent_batch(c4)
t3 = time.perf_counter()
print(f"import {1e3*(ti-t0):.1f} ms; first C4 {1e3*(t2-t1):.1f}; second C4 {1e3*(t3-t2):.1f}", flush=True)
