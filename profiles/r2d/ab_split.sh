#!/bin/bash
# A/B of the n <= 5 batch kernel's work split (PL_BATCH_SPLIT): the default library (even
# contiguous ranges) against build/variants/libpermlab_b200_nosplit.so (strided), bench.py's
# device-timed value for C1 and C2, interleaved repetitions on one box.
for rep in 1 2 3; do
  for cfg in c2 c1; do
    for lib in paper_1802_02779_b200/libpermlab_b200.so build/variants/libpermlab_b200_nosplit.so; do
      PL_NATIVE_LIB=$PWD/$lib python bench.py --config $cfg --no-suite --no-cpu --steps 50 --warmup 5 2>/dev/null |
        python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$lib'.split('/')[-1], 'us/step %.3f' % (1e3*d['ms_per_step']), 'frac %.3f' % d['roofline']['frac'], 'e2e %.1f M/s' % (d['e2e']['value']/1e6))"
    done
  done
done
