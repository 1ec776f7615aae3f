# C2 fused-kernel variants (device step time, L2 flushed), one line each
run() { echo "== $1"; shift; env "$@" python bench.py --config C2 --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  e2e %.1f us  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value']))
    elif 'Error' in l or 'error' in l: print(l)
"; }
run default X=1
run nsub2 PFB200_NSUB=2
run ept8 PFB200_EPT=8
run ept8_nst3 PFB200_EPT=8 PFB200_NST=3
run nst3 PFB200_NST=3
run default_again X=1
