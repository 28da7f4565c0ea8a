cd $GRAFT_REPO_ROOT
for c in 1 2 4 8; do
  for cfg in c3 c1; do
  PL_HOST_CHUNK_MB=$c python bench.py --config $cfg --steps 10 --warmup 3 --no-suite --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunk $c MB $cfg: e2e', round(d['e2e']['value']/1e6,2), 'M/s')" >> gpurun_out/chunk28.txt
  done
done
