"""Per-layer device time of one evaluation in a normal run (CUDA events between layers, no syncs)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1802_02779_b200 import configs
from paper_1802_02779_b200.sharded import device_hooks, sharded_layer_dp
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
a = torch.from_numpy(configs.generate(name)[0]).cuda()
layer_fn, top_fn = device_hooks(a)
for rep in range(3):
    evs = [torch.cuda.Event(enable_timing=True)]
    evs[0].record()
    def on_layer(k):
        e = torch.cuda.Event(enable_timing=True); e.record(); evs.append(e)
    v = sharded_layer_dp(a, 0, 1, layer_fn, top_fn, on_layer=on_layer)
    torch.cuda.synchronize()
    ts = [evs[i].elapsed_time(evs[i + 1]) for i in range(len(evs) - 1)]
    print(f"rep {rep}: total {sum(ts):.2f} ms;", " ".join(f"{k + 2}:{t:.2f}" for k, t in enumerate(ts) if t > 0.5))
