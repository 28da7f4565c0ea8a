cd $GRAFT_REPO_ROOT
python - >> gpurun_out/h2d24.txt 2>&1 <<'PY'
import torch, time
a = torch.empty(40_000_000 // 8, dtype=torch.float64).pin_memory(); d = torch.empty_like(a, device="cuda")
for _ in range(3): d.copy_(a, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): d.copy_(a, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("raw H2D 40 MB pinned: %.1f GB/s" % (10 * 40e6 / (e0.elapsed_time(e1) / 1e3) / 1e9))
PY
for c in 1 2 4 8 16; do
  PL_HOST_CHUNK_MB=$c python bench.py --config c2 --steps 10 --warmup 3 --no-suite --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunk $c MB: e2e', round(d['e2e']['value']/1e6,1), 'M/s')" >> gpurun_out/h2d24.txt
done
