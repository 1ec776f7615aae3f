# is the per-CTA setup bound by its (cold) code size?  task loop unrolled (default) vs one copy
for d in "" "PF_SETUP_QLOOP"; do
  echo "== $d"
  PFB200_DEFINES="PF_SETUP_TRACE;$d" python tools/trace_fused.py C2 2>&1 | grep "^setup" | tail -9
  PFB200_DEFINES="$d" python bench.py --config C2 --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step %.1f us kernel %.1f us value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['metric_value']))"
  PFB200_DEFINES="$d" python bench.py --config C1 --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C1 step %.1f us kernel %.1f us value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['metric_value']))"
done
