cd $GRAFT_REPO_ROOT
for i in 1 2 3; do
  for cfg in c3 c1 c2; do
  python bench.py --config $cfg --steps 10 --warmup 3 --no-suite --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$cfg: e2e', round(d['e2e']['value']/1e6,2), 'M/s value', round(d['value']/1e6,1))" >> gpurun_out/e2e29.txt
  done
done
