#!/bin/bash
# A/B of PL_FLAG_INPUT_READY in bench.py's graph-replayed batch steps (PL_BENCH_INPUT_READY=0: off).
for rep in 1 2 3; do
  for cfg in ${CFGS:-c2 c1}; do
    for on in 1 0; do
      PL_BENCH_INPUT_READY=$on python bench.py --config $cfg --no-suite --no-cpu --steps 50 --warmup 5 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', 'input_ready=$on', 'us/step %.3f' % (1e3*d['ms_per_step']), 'frac %.3f' % d['roofline']['frac'], 'e2e %.1f M/s' % (d['e2e']['value']/1e6))"
    done
  done
done
