cd $GRAFT_REPO_ROOT
for v in "" w2 w8 w16 nb2; do
  for c in c1 c2; do
    if [ -n "$v" ]; then export PL_NATIVE_LIB=profiles/_variants/$v.so; else unset PL_NATIVE_LIB; fi
    python bench.py --config $c --steps 20 --warmup 5 --no-suite --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$c', round(d['ms_per_step']*1000,2),'us', round(d['roofline']['frac'],3))" >> gpurun_out/geo16.txt 2>&1
  done
done
