#!/bin/bash
# A/B the event pass.  Each argument is a space-separated list of ENV=VALUE
# assignments, e.g.  "PFB200_NSUB=4"  or  "PFB200_DEFINES=PF_EXP_LIBDEVICE".
# Device timing (CUDA events, L2 flushed between steps) via bench.py.
for v in "$@"; do
  env $v python bench.py --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('%-50s step %6.1f us  event %6.1f us  frac %.3f nll %.17g' % ('$v' or 'default', d['ms_per_step']*1e3, r['kernel_ms']*1e3, r['frac'], d['nll']))"
done
