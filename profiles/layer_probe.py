"""Per-layer timing of the layer DP through pl_sz_layer (synchronising after each layer)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_1802_02779_b200 as pl
from paper_1802_02779_b200 import configs
from paper_1802_02779_b200.sharded import device_hooks, sharded_layer_dp
n = int(sys.argv[1]); dt = sys.argv[2]; fma = "--fma" in sys.argv
if dt == "c5":
    a = torch.from_numpy(configs.c5()).cuda()
else:
    import numpy as np
    a_np = configs.complex_uniform((n, n), seed=n) if dt == "c" else configs.uniform((n, n), seed=n)
    a = torch.from_numpy(a_np).cuda()
layer_fn, top_fn = device_hooks(a, fma=fma)
t = [time.perf_counter()]
def on_layer(k):
    torch.cuda.synchronize(); t.append(time.perf_counter())
    print(f"layer {k:2d}: {1000*(t[-1]-t[-2]):8.3f} ms", flush=True)
v = sharded_layer_dp(a, 0, 1, layer_fn, top_fn, on_layer=on_layer)
print("value", v)
