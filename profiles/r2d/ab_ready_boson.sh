#!/bin/bash
# A/B of PL_FLAG_INPUT_READY on the boson distribution steps of bench.py's suite (boson, boson_large).
for rep in 1 2 3; do
  for on in 1 0; do
    PL_BENCH_INPUT_READY=$on python bench.py --no-cpu --steps 20 --warmup 5 2>/dev/null |
      python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['suite']; print('input_ready=$on', 'boson us/step %.3f frac %.3f' % (1e3*s['boson']['ms_per_step'], s['boson']['roofline']['frac']), 'boson_large ms/step %.4f frac %.3f' % (s['boson_large']['ms_per_step'], s['boson_large']['roofline']['frac']))"
  done
done
