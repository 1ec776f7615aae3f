#!/bin/bash
# A/B the event kernel under PFB200_DEFINES variants (device timing via bench.py)
for v in "$@"; do
  PFB200_DEFINES="$v" python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('%-50s step %6.1f us  event %6.1f us  frac %.3f nll %.17g' % ('$v' or 'default', d['ms_per_step']*1e3, r['kernel_ms']*1e3, r['frac'], d['nll']))"
done
