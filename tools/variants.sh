#!/bin/bash
# A/B the event pass.  Each argument is a space-separated list of ENV=VALUE
# assignments, e.g.  "PFB200_NSUB=4"  or  "PFB200_DEFINES=PF_EXP_LIBDEVICE".
# Device timing (CUDA events, L2 flushed between steps) via bench.py;
# BENCH_ARGS adds bench options (e.g. "--config C3").
for v in "$@"; do
  env $v python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-fit $BENCH_ARGS 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print('%-50s step %8.1f us  event %8.1f us  frac %.3f value %.17g' % ('$v' or 'default', d['ms_per_step']*1e3, r['kernel_ms']*1e3, r['frac'], d['metric_value']))"
done
