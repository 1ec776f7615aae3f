run() { echo "== $1"; shift; env "$@" python bench.py --config C3 --steps 10 --warmup 3 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  frac %.3f  value %r' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['roofline']['frac'], d['metric_value']))
    elif 'Error' in l or 'error' in l: print(l)
"; }
run default X=1
run ept4_nst6 PFB200_EPT=4 PFB200_NST=6
run ept16_nst2 PFB200_EPT=16 PFB200_NST=2 PFB200_NSUB=8
run nsub8 PFB200_NSUB=8
run ept8_nst2 PFB200_NST=2
