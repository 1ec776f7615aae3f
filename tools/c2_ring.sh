# C2 ring depth vs stage size (fused kernel), device step and e2e; trace of the loop for each
run() { echo "== $1"; shift; env "$@" python bench.py --config C2 --steps 30 --warmup 5 --no-fit --no-cpu-baseline 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('step %.1f us  kernel %.1f us  e2e %.1f us  value %r fused=%s' % (d['ms_per_step']*1e3, d['roofline']['kernel_ms']*1e3, d['e2e']['ms_per_step']*1e3, d['metric_value'], d['roofline'].get('kernel')))
    elif 'Error' in l or 'error' in l: print(l)
"; }
run default X=1
run nst3 PFB200_NST=3
run ept8_nst4 PFB200_EPT=8 PFB200_NST=4
run ept8_nst6 PFB200_EPT=8 PFB200_NST=6
run ept4_nst8 PFB200_EPT=4 PFB200_NST=8
run default_again X=1
