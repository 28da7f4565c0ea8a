cd $GRAFT_REPO_ROOT
for v in 1 0 1 0; do
  for c in c1 c2; do
    PL_BATCH_PDL=$v python bench.py --config $c --steps 20 --warmup 5 --no-suite --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('pdl=$v', '$c', round(d['ms_per_step']*1000,2),'us', round(d['roofline']['frac'],3), round(d['e2e']['value']/1e6,1),'M/s e2e')" >> gpurun_out/pdl15.txt 2>&1
  done
done
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "c1 or c2 or small_orders or pipelined or torch_device or concurrent" >> gpurun_out/pdl15.txt 2>&1
