cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for u in 1 2 4; do
  for cm in 8 4 2; do
  PL_HOST_UP_STREAMS=$u PL_HOST_CHUNK_MB=$cm python bench.py --config c2 --steps 10 --warmup 3 --no-suite --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('up $u chunk $cm: C2 e2e', round(d['e2e']['value']/1e6,1), 'M/s')" >> gpurun_out/up31.txt
  done
done
python profiles/r2b/h2d_probe3.py >> gpurun_out/up31.txt
done
