# last-CTA arrival: fence + atomicAdd (default) vs one acq_rel atomic (PF_DONE_ACQREL)
run() { echo "== $1"; shift; env "$@" timeout 300 python bench.py --config C2 --steps 40 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.2f us  kernel %.2f us  e2e %.1f us  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value']))
"; }
for rep in 1 2 3; do
  run fence X=1
  run acqrel PFB200_DEFINES=PF_DONE_ACQREL
done
